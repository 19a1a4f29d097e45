"""ORACLE -- CPU restatement of the reference FV/RNS path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / the reported CPU baseline.
The product (paper_1901_10074_b200) never imports it.

It restates, function by function, the reference's algorithm
(/root/reference/pkg/src/hepack/ntt.py and fv.py) in numpy, with the
transform butterflies in plain C (oracle/ntt_ref.c, built by
__graft_entry__.build() into oracle/_build/libntt_oracle.so) in place of the
reference's numba kernel; a numpy stage loop is used when the C helper is
not built.  Parity is pinned by tests/test_oracle.py against golden vectors
generated from the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_SO = HERE / "_build" / "libntt_oracle.so"

SIGMA = 3.2
ERR_BOUND = 19
WORD_BITS = 30

_clib = None


def _c_helper():
    global _clib
    if _clib is None and _SO.exists():
        lib = C.CDLL(str(_SO))
        lib.oracle_ct_stages.restype = None
        lib.oracle_ct_stages.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                         C.c_void_p, C.c_int64]
        _clib = lib
    return _clib


# ---------------------------------------------------------------------------
# number theory (ntt.py:64-131)
# ---------------------------------------------------------------------------
def is_prime(n: int) -> bool:
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for s in small:
        if n % s == 0:
            return n == s
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def smallest_generator(p: int) -> int:
    m, fs, f = p - 1, [], 2
    while f * f <= m:
        if m % f == 0:
            fs.append(f)
            while m % f == 0:
                m //= f
        f = f + 1 if f == 2 else f + 2
    if m > 1:
        fs.append(m)
    g = 2
    while not all(pow(g, (p - 1) // q, p) != 1 for q in fs):
        g += 1
    return g


def ntt_primes(count: int, bits: int, two_n: int, below=None) -> list:
    p = ((1 << bits) // two_n) * two_n + 1
    if below is not None:
        p = min(p, ((below - 2) // two_n) * two_n + 1)
    out = []
    while len(out) < count:
        if p < two_n:
            raise ValueError("ran out of candidate primes")
        if is_prime(p):
            out.append(p)
        p -= two_n
    return out


def bit_reverse(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    return np.array([int(format(i, f"0{bits}b")[::-1], 2) for i in range(n)], dtype=np.int64)


# ---------------------------------------------------------------------------
# NTT over one prime (ntt.py:142-227)
# ---------------------------------------------------------------------------
class OracleNtt:
    """fwd(a)[k] = a(psi^(2k+1)), natural order; inv is its inverse."""

    def __init__(self, p: int, n: int):
        if (p - 1) % (2 * n):
            raise ValueError(f"p={p} is not 1 mod {2 * n}")
        self.p, self.n = p, n
        self.small = p < (1 << 31)
        self.dtype = np.int64 if self.small else object
        self.psi = pow(smallest_generator(p), (p - 1) // (2 * n), p)
        omega = self.psi * self.psi % p
        self.rev = bit_reverse(n)
        self.psi_pow = self._geometric(self.psi, n)
        self.ipsi_pow = self._geometric(pow(self.psi, p - 2, p), n)
        self.n_inv = pow(n, p - 2, p)
        self.fwd_stages = self._stage_tables(omega)
        self.inv_stages = self._stage_tables(pow(omega, p - 2, p))
        if self.small:
            self.fwd_flat = np.concatenate(self.fwd_stages).astype(np.int64)
            self.inv_flat = np.concatenate(self.inv_stages).astype(np.int64)
            self.fwd_sh = np.array([(int(w) << 32) // p for w in self.fwd_flat], dtype=np.int64)
            self.inv_sh = np.array([(int(w) << 32) // p for w in self.inv_flat], dtype=np.int64)

    def _geometric(self, base: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=self.dtype)
        acc = 1
        for i in range(count):
            out[i] = acc
            acc = acc * base % self.p
        return out

    def _stage_tables(self, w: int) -> list:
        tabs, half = [], 1
        while half < self.n:
            tabs.append(self._geometric(pow(w, self.n // (2 * half), self.p), half))
            half *= 2
        return tabs

    def _cyclic(self, a: np.ndarray, forward: bool) -> np.ndarray:
        p, n = self.p, self.n
        x = np.ascontiguousarray(a[..., self.rev])
        lib = _c_helper() if self.small else None
        if lib is not None:
            flat = np.ascontiguousarray(x.reshape(-1, n).astype(np.int64))
            tw, sh = (self.fwd_flat, self.fwd_sh) if forward else (self.inv_flat, self.inv_sh)
            lib.oracle_ct_stages(flat.ctypes.data, flat.shape[0], n, tw.ctypes.data,
                                 sh.ctypes.data, p)
            return flat.reshape(x.shape)
        lead = x.shape[:-1]
        tabs = self.fwd_stages if forward else self.inv_stages
        half = 1
        for tab in tabs:
            x = x.reshape(*lead, n // (2 * half), 2 * half)
            lo, hi = x[..., :half], x[..., half:] * tab % p
            x = np.concatenate(((lo + hi) % p, (lo - hi) % p), axis=-1).reshape(*lead, n)
            half *= 2
        return x

    def fwd(self, a) -> np.ndarray:
        a = np.asarray(a, dtype=self.dtype) % self.p
        return self._cyclic(a * self.psi_pow % self.p, True)

    def inv(self, ev) -> np.ndarray:
        ev = np.asarray(ev, dtype=self.dtype) % self.p
        a = self._cyclic(ev, False)
        return a * self.ipsi_pow % self.p * self.n_inv % self.p

    def negacyclic_mul(self, a, b) -> np.ndarray:
        return self.inv(self.fwd(a) * self.fwd(b) % self.p)


def schoolbook(a, b, n: int, p=None) -> np.ndarray:
    """Exact negacyclic product (ntt.py:230-245)."""
    a = [int(v) for v in a]
    b = [int(v) for v in b]
    out = [0] * n
    for i, x in enumerate(a):
        if x == 0:
            continue
        for j, y in enumerate(b):
            k = i + j
            if k < n:
                out[k] += x * y
            else:
                out[k - n] -= x * y
    res = np.array(out, dtype=object)
    return res % p if p is not None else res


class OracleCrt:
    """(k, n) residues <-> big integers (ntt.py:248-271)."""

    def __init__(self, primes):
        self.primes = list(primes)
        self.product = 1
        for p in self.primes:
            self.product *= p
        self.interp = np.array([(self.product // p) * pow(self.product // p, -1, p) % self.product
                                for p in self.primes], dtype=object)

    def to_big(self, res) -> np.ndarray:
        return res.astype(object).T @ self.interp % self.product

    def from_big(self, vals) -> np.ndarray:
        vals = np.asarray(vals, dtype=object)
        return np.stack([(vals % p).astype(np.int64) for p in self.primes])


# ---------------------------------------------------------------------------
# FV context, keys and operations (fv.py:45-432)
# ---------------------------------------------------------------------------
class OracleParams:
    def __init__(self, n: int, t: int, q_primes):
        if t % (2 * n) != 1:
            raise ValueError("plain modulus must be 1 mod 2n")
        self.n, self.t, self.q_primes, self.sigma = n, t, list(q_primes), SIGMA

    @classmethod
    def from_backend(cls, bp):
        count = max(2, -(-bp.coeff_modulus_bits // WORD_BITS))
        return cls(bp.ring_dimension, bp.plain_modulus,
                   ntt_primes(count, WORD_BITS, 2 * bp.ring_dimension))


class OracleContext:
    def __init__(self, fp: OracleParams):
        self.fp = fp
        n = self.n = fp.n
        self.t = fp.t
        self.q_ntt = [OracleNtt(p, n) for p in fp.q_primes]
        self.q_crt = OracleCrt(fp.q_primes)
        self.q = self.q_crt.product
        self.delta = self.q // self.t
        self.delta_mod = [self.delta % p for p in fp.q_primes]
        self.pcol = np.array(fp.q_primes, dtype=np.int64)[:, None]
        bits = n.bit_length() + 2 * self.q.bit_length() + 2
        self.aux_primes = ntt_primes(-(-bits // (WORD_BITS - 1)), WORD_BITS, 2 * n,
                                     below=min(fp.q_primes))
        self.aux_ntt = [OracleNtt(p, n) for p in self.aux_primes]
        self.aux_crt = OracleCrt(self.aux_primes)
        self.gadget = [(self.q // p) * pow(self.q // p, -1, p) % self.q for p in fp.q_primes]
        self.t_ntt = OracleNtt(self.t, n)
        e, exps = 1, []
        for _ in range(n // 2):
            exps.append(e)
            e = e * 3 % (2 * n)
        self.slot_to_ev = (np.array(exps, dtype=np.int64) - 1) // 2

    # samplers: the reference's exact Generator calls (fv.py:114-129)
    def rand_uniform(self, rng):
        return np.stack([rng.integers(0, p, self.n, dtype=np.int64) for p in self.fp.q_primes])

    def rand_ternary(self, rng):
        return rng.integers(-1, 2, self.n, dtype=np.int64)

    def rand_error(self, rng):
        e = np.rint(rng.normal(0.0, self.fp.sigma, self.n)).astype(np.int64)
        return np.clip(e, -ERR_BOUND, ERR_BOUND)

    def rns(self, small):
        return np.asarray(small, dtype=np.int64) % self.pcol

    def ring_mul(self, a, b):
        return np.stack([tr.negacyclic_mul(a[i], b[i]) for i, tr in enumerate(self.q_ntt)])

    def galois(self, a, g: int):
        j = np.arange(self.n, dtype=np.int64)
        idx = j * g % (2 * self.n)
        out = np.zeros_like(a)
        out[..., idx % self.n] = a * np.where(idx < self.n, 1, -1)
        return out % self.pcol


class OracleSwitchKey:
    def __init__(self, body, mask):
        self.body, self.mask = body, mask


class OracleKeys:
    def __init__(self, context, secret, public, relin, galois):
        self.context, self.secret, self.public = context, secret, public
        self.relin, self.galois = relin, galois


def switch_key(ctx: OracleContext, s, target, rng) -> OracleSwitchKey:
    k = len(ctx.fp.q_primes)
    bodies, masks = [], []
    for i in range(k):
        a = ctx.rand_uniform(rng)
        e = ctx.rns(ctx.rand_error(rng))
        gi = np.array([ctx.gadget[i] % p for p in ctx.fp.q_primes], dtype=np.int64)[:, None]
        body = (-(ctx.ring_mul(a, s) + e) % ctx.pcol + target * gi % ctx.pcol) % ctx.pcol
        bodies.append(body)
        masks.append(a)
    body = [tr.fwd(np.stack([bodies[i][j] for i in range(k)])) for j, tr in enumerate(ctx.q_ntt)]
    mask = [tr.fwd(np.stack([masks[i][j] for i in range(k)])) for j, tr in enumerate(ctx.q_ntt)]
    return OracleSwitchKey(body, mask)


def switch_key_wide(primes, n, s_rns, target_rns, rng) -> OracleSwitchKey:
    """_keyswitch_key (fv.py:176-202) for any prime width: the same Generator
    calls as the reference's _FvContext samplers (fv.py:114-129), the ring
    products and the gadget scalars in object arithmetic, as the reference's
    object-dtype path computes them for p >= 2^31."""
    q = 1
    for p in primes:
        q *= p
    gadget = [(q // p) * pow(q // p, -1, p) % q for p in primes]
    ntts = [OracleNtt(p, n) for p in primes]
    pcol = np.array(primes, dtype=object)[:, None]
    k = len(primes)
    bodies, masks = [], []
    for i in range(k):
        a = np.stack([rng.integers(0, p, n, dtype=np.int64) for p in primes])
        e = np.clip(np.rint(rng.normal(0.0, SIGMA, n)).astype(np.int64), -ERR_BOUND, ERR_BOUND)
        e = e.astype(object) % pcol
        prod = np.stack([tr.negacyclic_mul(a[j], s_rns[j]) for j, tr in enumerate(ntts)])
        g = np.array([gadget[i] % p for p in primes], dtype=object)[:, None]
        body = (-((prod + e) % pcol) % pcol + np.asarray(target_rns, dtype=object) * g % pcol) % pcol
        bodies.append(body)
        masks.append(a.astype(object))
    body = [tr.fwd(np.stack([bodies[i][j] for i in range(k)])) for j, tr in enumerate(ntts)]
    mask = [tr.fwd(np.stack([masks[i][j] for i in range(k)])) for j, tr in enumerate(ntts)]
    return OracleSwitchKey(body, mask)


def ks64_case(primes, n, seed):
    """Config-4 key-switch case drawn like make_golden.gen_ks64 draws it from
    the reference: secret s (ternary), target s^2, the switch key, then the
    input polynomial c uniform mod each prime -- one Generator."""
    rng = np.random.default_rng(seed)
    ntts = [OracleNtt(p, n) for p in primes]
    pcol = np.array(primes, dtype=object)[:, None]
    s = rng.integers(-1, 2, n, dtype=np.int64).astype(object) % pcol
    target = np.stack([tr.negacyclic_mul(s[j], s[j]) for j, tr in enumerate(ntts)])
    key = switch_key_wide(primes, n, s, target, rng)
    c = np.stack([rng.integers(0, p, n, dtype=np.int64) for p in primes])
    return key, c


def keyswitch(ctx: OracleContext, c, key: OracleSwitchKey):
    k = len(ctx.fp.q_primes)
    d0 = np.empty((k, ctx.n), dtype=np.int64)
    d1 = np.empty((k, ctx.n), dtype=np.int64)
    for j, tr in enumerate(ctx.q_ntt):
        dig = tr.fwd(c % tr.p)
        s0 = (dig * key.body[j] % tr.p).sum(axis=0) % tr.p
        s1 = (dig * key.mask[j] % tr.p).sum(axis=0) % tr.p
        d0[j], d1[j] = tr.inv(np.stack([s0, s1]))
    return d0, d1


def keygen(fp: OracleParams, rotation_offsets=None, rng=None) -> OracleKeys:
    rng = rng if rng is not None else np.random.default_rng()
    ctx = OracleContext(fp)
    s = ctx.rns(ctx.rand_ternary(rng))
    a = ctx.rand_uniform(rng)
    e = ctx.rns(ctx.rand_error(rng))
    pk = ((-(ctx.ring_mul(a, s) + e)) % ctx.pcol, a)
    relin = switch_key(ctx, s, ctx.ring_mul(s, s), rng)
    half = fp.n // 2
    offs = {1 << j for j in range((half - 1).bit_length())}
    if rotation_offsets:
        offs |= {o % half for o in rotation_offsets if o % half}
    galois = {off: switch_key(ctx, s, ctx.galois(s, pow(3, off, 2 * fp.n)), rng)
              for off in sorted(offs)}
    return OracleKeys(ctx, s, pk, relin, galois)


class OracleCiphertext:
    __slots__ = ("parts", "level_used", "params", "_live")

    def __init__(self, parts, level_used, params):
        self.parts, self.level_used, self.params, self._live = parts, level_used, params, True


def make_backend_class():
    """OracleFvBackend, built on the package's SlotBackend contract (host
    bookkeeping only) so the serial layer_eval/infer can drive it."""
    from paper_1901_10074_b200.engine import SlotBackend
    from paper_1901_10074_b200.errors import ParamMismatchError

    class OracleFvBackend(SlotBackend):
        def __init__(self, params, keys=None, rng=None):
            if params.slot_count != params.ring_dimension // 2:
                raise ParamMismatchError("FV backend requires slot_count = n/2")
            super().__init__(params)
            self.rng = rng if rng is not None else np.random.default_rng()
            if keys is None:
                keys = keygen(OracleParams.from_backend(params), rng=self.rng)
            self.keys = keys
            self.ctx = ctx = keys.context
            if ctx.t != params.plain_modulus or ctx.n != params.ring_dimension:
                raise ParamMismatchError("key set was generated for different parameters")
            self._s = [tr.fwd(keys.secret[j]) for j, tr in enumerate(ctx.q_ntt)]
            s2 = ctx.ring_mul(keys.secret, keys.secret)
            self._s2 = [tr.fwd(s2[j]) for j, tr in enumerate(ctx.q_ntt)]
            self._pk = tuple([tr.fwd(part[j]) for j, tr in enumerate(ctx.q_ntt)]
                             for part in keys.public)

        def encode(self, vec):
            ctx = self.ctx
            ev = np.zeros(ctx.n, dtype=ctx.t_ntt.dtype)
            ev[ctx.slot_to_ev] = np.asarray(vec, dtype=ctx.t_ntt.dtype) % ctx.t
            return ctx.t_ntt.inv(ev)

        def decode(self, poly):
            return self.ctx.t_ntt.fwd(poly)[self.ctx.slot_to_ev]

        def centred(self, poly):
            t = self.ctx.t
            m = np.asarray(poly) % t
            return np.where(m > t // 2, m - t, m)

        def delta_m(self, m):
            ctx = self.ctx
            if ctx.t < (1 << 31):
                m = np.asarray(m, dtype=np.int64)
                return np.stack([m % p * ctx.delta_mod[i] % p
                                 for i, p in enumerate(ctx.fp.q_primes)])
            m = np.asarray(m, dtype=object)
            return np.stack([(m * ctx.delta_mod[i] % p).astype(np.int64)
                             for i, p in enumerate(ctx.fp.q_primes)])

        def _ct(self, parts, level):
            return OracleCiphertext(parts, level, self.params)

        def _encrypt(self, vec):
            ctx = self.ctx
            u = ctx.rns(ctx.rand_ternary(self.rng))
            e1 = ctx.rns(ctx.rand_error(self.rng))
            e2 = ctx.rns(ctx.rand_error(self.rng))
            dm = self.delta_m(self.encode(vec))
            c0 = np.empty((len(ctx.q_ntt), ctx.n), dtype=np.int64)
            c1 = np.empty_like(c0)
            for j, tr in enumerate(ctx.q_ntt):
                ue = tr.fwd(u[j])
                pair = tr.inv(np.stack([ue * self._pk[0][j] % tr.p, ue * self._pk[1][j] % tr.p]))
                c0[j] = (pair[0] + e1[j] + dm[j]) % tr.p
                c1[j] = (pair[1] + e2[j]) % tr.p
            return self._ct([c0, c1], 0)

        def decrypt_poly(self, ct):
            ctx = self.ctx
            sk = [self._s, self._s2]
            acc = ct.parts[0].copy()
            for j, tr in enumerate(ctx.q_ntt):
                evs = tr.fwd(np.stack([c[j] for c in ct.parts[1:]]))
                tot = np.zeros(ctx.n, dtype=np.int64)
                for m in range(evs.shape[0]):
                    tot = (tot + evs[m] * sk[m][j] % tr.p) % tr.p
                acc[j] = (acc[j] + tr.inv(tot)) % tr.p
            x = ctx.q_crt.to_big(acc)
            return (x * ctx.t + ctx.q // 2) // ctx.q % ctx.t

        def _decrypt(self, ct):
            return np.asarray(self.decode(self.decrypt_poly(ct)), dtype=self._dtype)

        def _add(self, a, b, level):
            return self._ct([(x + y) % self.ctx.pcol for x, y in zip(a.parts, b.parts)], level)

        def _add_plain(self, a, vec, level):
            dm = self.delta_m(self.encode(vec))
            return self._ct([(a.parts[0] + dm) % self.ctx.pcol] + [p.copy() for p in a.parts[1:]],
                            level)

        def _cmult(self, a, vec, level):
            ctx = self.ctx
            m = self.centred(self.encode(vec))
            out = [np.empty((len(ctx.q_ntt), ctx.n), dtype=np.int64) for _ in a.parts]
            for j, tr in enumerate(ctx.q_ntt):
                me = tr.fwd(m % tr.p)
                prods = tr.inv(tr.fwd(np.stack([c[j] for c in a.parts])) * me % tr.p)
                for c in range(len(a.parts)):
                    out[c][j] = prods[c]
            return self._ct(out, level)

        def tensor(self, a, b):
            ctx = self.ctx
            hq = ctx.q // 2
            lifted = []
            for c in (a.parts[0], a.parts[1], b.parts[0], b.parts[1]):
                x = ctx.q_crt.to_big(c)
                lifted.append(ctx.aux_crt.from_big(np.where(x > hq, x - ctx.q, x)))
            na = len(ctx.aux_primes)
            t0, t1, t2 = (np.empty((na, ctx.n), dtype=np.int64) for _ in range(3))
            for i, tr in enumerate(ctx.aux_ntt):
                ev = tr.fwd(np.stack([r[i] for r in lifted]))
                t0[i], t1[i], t2[i] = tr.inv(np.stack([
                    ev[0] * ev[2] % tr.p, (ev[0] * ev[3] + ev[1] * ev[2]) % tr.p,
                    ev[1] * ev[3] % tr.p]))
            ha = ctx.aux_crt.product // 2
            out = []
            for st in (t0, t1, t2):
                x = ctx.aux_crt.to_big(st)
                x = np.where(x > ha, x - ctx.aux_crt.product, x)
                out.append(ctx.q_crt.from_big((x * ctx.t + ctx.q // 2) // ctx.q % ctx.q))
            return out

        def _mult(self, a, b, level):
            t0, t1, t2 = self.tensor(a, b)
            d0, d1 = keyswitch(self.ctx, t2, self.keys.relin)
            return self._ct([(t0 + d0) % self.ctx.pcol, (t1 + d1) % self.ctx.pcol], level)

        def rotation_hops(self, offset):
            if offset == 0:
                return []
            if offset in self.keys.galois:
                return [offset]
            return [1 << j for j in range(offset.bit_length()) if offset >> j & 1]

        def _rotate(self, a, offset, level):
            if offset == 0:
                return self._ct([p.copy() for p in a.parts], level)
            ctx = self.ctx
            parts = a.parts
            for off in self.rotation_hops(offset):
                g = pow(3, off, 2 * ctx.n)
                p0, p1 = ctx.galois(parts[0], g), ctx.galois(parts[1], g)
                d0, d1 = keyswitch(ctx, p1, self.keys.galois[off])
                parts = [(p0 + d0) % ctx.pcol, d1]
            return self._ct(parts, level)

    return OracleFvBackend


_BACKEND_CLS = None


def OracleFvBackend(params, keys=None, rng=None):  # noqa: N802 - factory with class-like name
    global _BACKEND_CLS
    if _BACKEND_CLS is None:
        _BACKEND_CLS = make_backend_class()
    return _BACKEND_CLS(params, keys=keys, rng=rng)


def limb_digest(parts) -> str:
    """sha256 over the int64 little-endian bytes of each (k, n) stack."""
    import hashlib

    h = hashlib.sha256()
    for p in parts:
        h.update(np.ascontiguousarray(np.asarray(p, dtype=np.int64)).astype("<i8").tobytes())
    return h.hexdigest()
