"""Fan-Vercauteren over RNS, device-resident: the GPU drop-in for the
reference's ``hepack.fv`` (/root/reference/pkg/src/hepack/fv.py).

Same public surface -- ``FvParams``, ``SwitchKey``, ``KeySet``, ``keygen``,
``FvCiphertext``, ``FvBackend``, ``run_sequence``, ``fv_conformance`` -- and
bit-identical results: keys and encryption randomness are drawn on the host
through the caller's ``numpy.random.Generator`` with exactly the reference's
calls and order (fv.py:114-129, 231-251, 317-321); everything else (NTTs,
key generation arithmetic, encryption, decryption rounding, ct x pt, exact
ct x ct tensor + relinearisation, Galois key switching) runs in libhefv.so.

Ciphertexts live in HBM as (parts, k, N) uint32 stacks; ``FvCiphertext.parts``
downloads lazily to the reference's list of (k, N) int64 arrays.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .engine import SlotBackend
from .errors import FormatError, ParamMismatchError
from .params import BackendParams
from .ring import (
    WORD_BITS,
    CrtConstants,
    bitrev_perm,
    find_ntt_primes,
    gadget,
    galois_element,
    root_of_unity,
    slot_to_eval,
)

# The aux-basis key switch's three NTT primes are the largest below
# 2^28 (1 + 1/16): above 2^28 (valid lazy inputs, Montgomery bound) and close
# enough to it that ks_aux.cu takes the CRT quotient terms by a shift.
KS_AUX_BELOW = (1 << 28) + (1 << 24)

SIGMA = 3.2
ERR_BOUND = 19  # 6-sigma truncation (fv.py:25-26)


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# parameters
# ---------------------------------------------------------------------------
@dataclass
class FvParams:
    """n, t and the q primes (fv.py:45-64)."""

    n: int
    t: int
    q_primes: list
    sigma: float = SIGMA

    def __post_init__(self):
        if self.t % (2 * self.n) != 1:
            raise ValueError(
                f"plain_modulus {self.t} must be 1 mod 2n={2 * self.n} for batching")

    @classmethod
    def from_backend(cls, params: BackendParams) -> "FvParams":
        count = max(2, -(-params.coeff_modulus_bits // WORD_BITS))
        primes = find_ntt_primes(count, WORD_BITS, 2 * params.ring_dimension)
        return cls(n=params.ring_dimension, t=params.plain_modulus, q_primes=primes)


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class FvContext:
    """Constants of one parameter set, mirrored on the device.

    Host attributes follow _FvContext (fv.py:75-110): n, t, q, delta,
    delta_mod, aux_primes, gadget, slot_to_ev, fp.  ``q_ntt``/``aux_ntt``/
    ``t_ntt`` are GPU ``NttPrime`` objects created on first use."""

    def __init__(self, fp: FvParams):
        import ctypes as C

        nat.require_device()
        lib = nat.load()
        torch = _torch()
        self.fp = fp
        self.n = n = fp.n
        self.log_n = n.bit_length() - 1
        if self.log_n > 14:
            raise ValueError("the FV kernels support ring dimensions up to 2^14")
        self.t = fp.t
        self.q_primes = list(fp.q_primes)
        self.k = len(self.q_primes)
        self.pcol = np.array(self.q_primes, dtype=np.int64)[:, None]
        qc = CrtConstants.build(self.q_primes)
        self.q = qc.product
        if self.q < 1 << 32:
            # the exact t/q roundings run Knuth D on >= 2 words (hefv_fv_setup)
            raise ParamMismatchError("the GPU backend needs q >= 2^32 (two or more q primes)")
        self.delta = self.q // fp.t
        self.delta_mod = [self.delta % p for p in self.q_primes]
        need_bits = n.bit_length() + 2 * self.q.bit_length() + 2
        count = -(-need_bits // (WORD_BITS - 1))
        self.aux_primes = find_ntt_primes(count, WORD_BITS, 2 * n, below=min(self.q_primes))
        self.a = len(self.aux_primes)
        mc = CrtConstants.build(self.aux_primes)
        self.gadget = gadget(self.q_primes)
        self.slot_to_ev = slot_to_eval(n)
        if fp.t >= 1 << 62:
            raise ValueError("plain modulus must be below 2^62")
        # three ~28-bit primes for the aux-basis key switch (ks_aux.cu): used
        # when it needs fewer transforms than the per-prime one (k > 8)
        import os

        self.ks_aux = (8 < self.k <= 24 and 10 <= self.log_n <= 14
                       and os.environ.get("HEFV_KS_AUX", "1") != "0")
        self.ks_aux_primes = (find_ntt_primes(3, 29, 2 * n, below=KS_AUX_BELOW)
                              if self.ks_aux else [])
        primes32 = self.q_primes + self.aux_primes + self.ks_aux_primes
        psi32 = [root_of_unity(p, n) for p in primes32]
        psi_t = root_of_unity(fp.t, n)
        arr32 = (C.c_uint32 * len(primes32))(*primes32)
        apsi32 = (C.c_uint32 * len(primes32))(*psi32)
        arr64 = (C.c_uint64 * 1)(fp.t)
        apsi64 = (C.c_uint64 * 1)(psi_t)
        h = C.c_void_p()
        nat.check(lib.hefv_ctx_create(C.byref(h), self.log_n, len(primes32), arr32, apsi32, 1,
                                      arr64, apsi64), "hefv_ctx_create")
        self._h = h
        self._lib = lib

        def cbuf(a, ctype):
            a = np.ascontiguousarray(a)
            return a.ctypes.data_as(C.POINTER(ctype)), a

        keep = []

        def c32(a):
            p, arr = cbuf(np.asarray(a, dtype=np.uint32), C.c_uint32)
            keep.append(arr)
            return p

        s2e = np.ascontiguousarray(self.slot_to_ev.astype(np.int32))
        keep.append(s2e)
        nat.check(lib.hefv_fv_setup(
            h, self.k, self.a, 0, s2e.ctypes.data_as(C.POINTER(C.c_int32)),
            qc.words, c32(qc.prod_words), c32(qc.half_words), c32(qc.hat_words.reshape(-1)),
            c32(qc.hat_inv), mc.words, c32(mc.prod_words), c32(mc.half_words),
            c32(mc.hat_words.reshape(-1)), c32(mc.hat_inv), c32(self.delta_mod)),
            "hefv_fv_setup")
        if self.ks_aux:
            nat.check(lib.hefv_ks_aux_setup(h, self.k + self.a), "hefv_ks_aux_setup")
        # everything the three setup calls received, for hosts that drive the
        # C-ABI without this module (tests/c_host)
        self.setup_record = {
            "log_n": self.log_n, "primes32": primes32, "psi32": psi32, "primes64": [fp.t],
            "psi64": [psi_t], "k": self.k, "a": self.a, "t_index": 0, "slot_to_ev": s2e,
            "wq": qc.words, "q": qc.prod_words, "qhalf": qc.half_words,
            "qhat": qc.hat_words.reshape(-1), "qhat_inv": qc.hat_inv, "wm": mc.words,
            "m": mc.prod_words, "mhalf": mc.half_words, "mhat": mc.hat_words.reshape(-1),
            "mhat_inv": mc.hat_inv, "delta_mod": self.delta_mod,
            "ks_aux_base": self.k + self.a if self.ks_aux else -1}
        # gadget_i mod q_j table (k x k)
        gtab = np.array([[g % p for p in self.q_primes] for g in self.gadget], dtype=np.int64)
        self.d_gadget = nat.to_device(gtab.astype(np.int32))
        self.p_col = np.array(self.q_primes, dtype=np.int64)[:, None]
        self.brev = bitrev_perm(self.log_n)
        self._ntt_cache = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and nat._lib is not None:
            nat._lib.hefv_ctx_destroy(h)
            self._h = None

    # ---- reference-compatible transform objects (lazy) ----
    def _ntt(self, p):
        from .ntt import NttPrime

        tr = self._ntt_cache.get(p)
        if tr is None:
            tr = self._ntt_cache[p] = NttPrime(p, self.n)
        return tr

    @property
    def q_ntt(self):
        return [self._ntt(p) for p in self.q_primes]

    @property
    def aux_ntt(self):
        return [self._ntt(p) for p in self.aux_primes]

    @property
    def t_ntt(self):
        return self._ntt(self.t)

    # ---- host samplers: identical Generator calls (fv.py:114-129) ----
    def rand_uniform(self, rng) -> np.ndarray:
        return np.stack([rng.integers(0, p, self.n, dtype=np.int64) for p in self.q_primes])

    def rand_ternary(self, rng) -> np.ndarray:
        return rng.integers(-1, 2, self.n, dtype=np.int64)

    def rand_error(self, rng) -> np.ndarray:
        e = np.rint(rng.normal(0.0, self.fp.sigma, self.n)).astype(np.int64)
        return np.clip(e, -ERR_BOUND, ERR_BOUND)

    def to_rns(self, small) -> np.ndarray:
        return np.asarray(small, dtype=np.int64) % self.p_col

    def galois_small(self, small: np.ndarray, g: int) -> np.ndarray:
        """x -> x^g on a small signed host polynomial (fv.py:157-173)."""
        j = np.arange(self.n, dtype=np.int64)
        idx = j * g % (2 * self.n)
        out = np.zeros(self.n, dtype=np.int64)
        out[idx % self.n] = np.where(idx < self.n, small, -small)
        return out

    # ---- device helpers ----
    def empty(self, *shape, dtype=None):
        torch = _torch()
        return torch.empty(shape, dtype=dtype or torch.int32, device="cuda")

    def call(self, name, *args):
        nat.call(name, self._h, *args)

    def stream(self):
        return nat.stream_handle()

    def small_to_ntt(self, small: np.ndarray, montgomery=False):
        """(B, N) signed small ints -> (B, k, N) NTT (device order)."""
        torch = _torch()
        s = np.asarray(small, dtype=np.int8).reshape(-1, self.n)
        d = nat.to_device(s)
        out = self.empty(s.shape[0], self.k, self.n)
        self.call("hefv_small_to_rns", d.data_ptr(), out.data_ptr(), s.shape[0], 1,
                  1 if montgomery else 0, self.stream())
        return out

    def upload_residues(self, arr: np.ndarray):
        torch = _torch()
        return nat.to_device(np.asarray(arr, dtype=np.int64).astype(np.int32))

    def ntt_q(self, stacks, inverse=False, natural=False):
        """In-device transform of (B, k, N) stacks under the q primes."""
        out = _torch().empty_like(stacks)
        b = stacks.numel() // (self.k * self.n)
        self.call("hefv_ntt_inv32" if inverse else "hefv_ntt_fwd32", stacks.data_ptr(),
                  out.data_ptr(), b, self.k, 0, 1 if natural else 0, self.stream())
        return out

    def elementwise(self, op, a, b, c=None, b_rows=None, c_rows=None):
        out = _torch().empty_like(a)
        rows = a.numel() // (self.k * self.n)
        br = b_rows if b_rows is not None else b.numel() // (self.k * self.n)
        cr = (c_rows if c_rows is not None else c.numel() // (self.k * self.n)) if c is not None else 1
        self.call("hefv_elementwise", op, a.data_ptr(), b.data_ptr(), nat.ptr(c),
                  out.data_ptr(), rows, br, cr, self.stream())
        return out

    def mont_inv_rows(self):
        """(1, k, N) stack holding 2^-32 mod p_j in row j (leaves Montgomery form)."""
        if getattr(self, "_mont_inv", None) is None:
            v = np.array([pow(1 << 32, -1, p) for p in self.q_primes], dtype=np.int64)
            self._mont_inv = nat.to_device(
                np.repeat(v[:, None], self.n, axis=1).astype(np.int32)[None])
        return self._mont_inv

    def to_mont(self, a):
        out = _torch().empty_like(a)
        self.call("hefv_to_montgomery", a.data_ptr(), out.data_ptr(),
                  a.numel() // (self.k * self.n), self.stream())
        return out

    def dev_to_natural(self, stacks_dev_order) -> np.ndarray:
        """Host copy of device-order NTT stacks in the reference's natural order."""
        host = nat.to_host(stacks_dev_order).astype(np.int64)
        out = np.empty_like(host)
        out[..., self.brev] = host
        return out

    def natural_to_dev(self, stacks_natural: np.ndarray) -> np.ndarray:
        return np.asarray(stacks_natural)[..., self.brev]


# ---------------------------------------------------------------------------
# keys
# ---------------------------------------------------------------------------
class SwitchKey:
    """Key-switch material, device-resident (fv.py:67-72).

    ``body_dev``/``mask_dev``: (k, k, N) [target prime j][digit i], device NTT
    order, Montgomery form.  ``body``/``mask`` give the reference's layout
    (list over j of (k, N) natural-order int64) on demand."""

    def __init__(self, ctx: FvContext, body_dev, mask_dev):
        self._ctx = ctx
        self.body_dev = body_dev
        self.mask_dev = mask_dev
        # aux-basis form for hefv_keyswitch_aux (the tensor-core contraction's
        # per-point key operands; hefv_ks_aux_key_words)
        self.aux_dev = None
        if ctx.ks_aux:
            import ctypes as C

            torch = _torch()
            words = C.c_int64()
            ctx.call("hefv_ks_aux_key_words", C.byref(words))
            self.aux_dev = torch.empty(words.value, dtype=torch.int32, device="cuda")
            ctx.call("hefv_ks_aux_key", body_dev.data_ptr(), mask_dev.data_ptr(),
                     self.aux_dev.data_ptr(), ctx.stream())
        self._handle = None

    @property
    def handle(self):
        """The C-ABI ``hefv_key*`` over this key's device buffers
        (hefv_key_wrap; the tensors stay owned by this object)."""
        if self._handle is None:
            import ctypes as C

            h = C.c_void_p()
            aux = self.aux_dev.data_ptr() if self.aux_dev is not None else None
            self._ctx.call("hefv_key_wrap", self.body_dev.data_ptr(), self.mask_dev.data_ptr(),
                           aux, C.byref(h))
            self._handle = h
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and nat._lib is not None:
            nat._lib.hefv_key_free(h)
            self._handle = None

    def _host(self, dev):
        """Device layout -> reference layout: Montgomery form undone on the
        device (x * (2^-32 mod p_j) mod p_j), then the device NTT order
        permuted back to natural order on download."""
        ctx = self._ctx
        # (j, i, N) -> (i, j, N): every digit row i is a stack over the primes j
        t = dev.transpose(0, 1).contiguous()
        plain = ctx.elementwise(2, t, ctx.mont_inv_rows(), b_rows=1).transpose(0, 1)
        host = nat.to_host(plain.contiguous()).astype(np.int64)
        out = []
        for j in range(ctx.k):
            nat_order = np.empty_like(host[j])
            nat_order[..., ctx.brev] = host[j]
            out.append(nat_order)
        return out

    @classmethod
    def from_host(cls, ctx: FvContext, body, mask) -> "SwitchKey":
        """Upload a key in the reference's stored form (list over target prime
        j of (k, N) natural-order NTT values, fv.py:67-72) into the device
        layout used by the key-switch kernel: residues checked and permuted to
        device order on the host, Montgomery form entered on the device."""

        def dev(stacks):
            if len(stacks) != ctx.k or any(np.shape(s) != (ctx.k, ctx.n) for s in stacks):
                raise FormatError("switch key does not match the parameter set")
            arr = np.empty((ctx.k, ctx.k, ctx.n), dtype=np.int64)
            for j, p in enumerate(ctx.q_primes):
                x = ctx.natural_to_dev(np.asarray(stacks[j], dtype=np.int64))
                if (x < 0).any() or (x >= p).any():
                    raise FormatError("switch key residue outside [0, p_j)")
                arr[j] = x
            d = nat.to_device(arr.astype(np.int32))            # (j, i, N)
            t = d.transpose(0, 1).contiguous()                   # (i, j, N)
            return ctx.to_mont(t).transpose(0, 1).contiguous()   # back to (j, i, N)

        return cls(ctx, dev(body), dev(mask))

    @property
    def body(self):
        return self._host(self.body_dev)

    @property
    def mask(self):
        return self._host(self.mask_dev)


@dataclass
class KeySet:
    """Secret/public/evaluation keys plus the shared context (fv.py:220-228)."""

    context: FvContext
    secret_small: np.ndarray
    pk_ntt: object          # (2, k, N) device order, canonical
    relin: SwitchKey
    galois: dict
    s_ntt: object = None    # (k, N) canonical device order
    _cache: dict = field(default_factory=dict)

    @classmethod
    def from_host(cls, ctx: FvContext, secret, public, relin, galois) -> "KeySet":
        """Key set from the reference's stored form (serialize.read_keyset):
        secret (k, N) residues, public coefficient pair, and (body, mask)
        lists per switch key."""
        secret = np.asarray(secret, dtype=np.int64)
        if secret.shape != (ctx.k, ctx.n):
            raise FormatError("secret key does not match the parameter set")
        p0 = ctx.q_primes[0]
        small = np.where(secret[0] > p0 // 2, secret[0] - p0, secret[0])
        if np.abs(small).max(initial=0) > 1 or not np.array_equal(ctx.to_rns(small), secret):
            raise FormatError("secret key is not ternary")
        s_ntt = ctx.small_to_ntt(small)[0]
        pk = np.stack([np.asarray(x, dtype=np.int64) for x in public])
        pk_ntt = ctx.ntt_q(ctx.upload_residues(pk))
        keys = cls(context=ctx, secret_small=small.astype(np.int8), pk_ntt=pk_ntt,
                   relin=SwitchKey.from_host(ctx, *relin),
                   galois={int(off): SwitchKey.from_host(ctx, *bm) for off, bm in galois.items()},
                   s_ntt=s_ntt)
        keys._cache["public"] = (pk[0], pk[1])
        return keys

    @property
    def secret(self) -> np.ndarray:
        return self.context.to_rns(self.secret_small)

    @property
    def public(self) -> tuple:
        """(pk0, pk1) coefficient stacks, as the reference stores them."""
        if "public" not in self._cache:
            ctx = self.context
            coeff = ctx.ntt_q(self.pk_ntt.contiguous(), inverse=True)
            host = nat.to_host(coeff).astype(np.int64)
            self._cache["public"] = (host[0], host[1])
        return self._cache["public"]


def _switch_key(ctx: FvContext, s_ntt, target_ntt, rng) -> SwitchKey:
    """Digit keys switching ``target`` back to ``s`` (fv.py:176-202); the
    Generator is consumed digit by digit exactly as the reference does."""
    torch = _torch()
    k, n = ctx.k, ctx.n
    body = torch.empty((k, k, n), dtype=torch.int32, device="cuda")
    mask = torch.empty_like(body)
    st = ctx.stream()
    for i in range(k):
        a = ctx.rand_uniform(rng)
        e = ctx.rand_error(rng)
        a_d = nat.to_device(a.astype(np.int32))
        e_d = nat.to_device(e.astype(np.int8))
        ctx.call("hefv_keygen_digit", a_d.data_ptr(), e_d.data_ptr(), i,
                 ctx.d_gadget[i].data_ptr(), s_ntt.data_ptr(), target_ntt.data_ptr(),
                 body.data_ptr(), mask.data_ptr(), st)
    return SwitchKey(ctx, body, mask)


def keygen(fp: FvParams, rotation_offsets=None, rng=None) -> KeySet:
    """Generate keys (fv.py:231-251) with the same Generator stream."""
    rng = rng if rng is not None else np.random.default_rng()
    ctx = FvContext(fp)
    s = ctx.rand_ternary(rng)
    a = ctx.rand_uniform(rng)
    e = ctx.rand_error(rng)
    s_ntt = ctx.small_to_ntt(s)[0]
    a_ntt = ctx.ntt_q(ctx.upload_residues(a)[None])[0]
    e_ntt = ctx.small_to_ntt(e)[0]
    pk0 = ctx.elementwise(3, a_ntt, s_ntt, e_ntt)  # -(a s + e)
    pk_ntt = _torch().stack([pk0, a_ntt])
    s2_ntt = ctx.elementwise(2, s_ntt, s_ntt)
    relin = _switch_key(ctx, s_ntt, s2_ntt, rng)
    half = fp.n // 2
    offsets = {1 << j for j in range((half - 1).bit_length())}
    if rotation_offsets:
        offsets |= {off % half for off in rotation_offsets if off % half}
    galois = {}
    for off in sorted(offsets):
        g = galois_element(off, fp.n)
        tgt = ctx.small_to_ntt(ctx.galois_small(s, g))[0]
        galois[off] = _switch_key(ctx, s_ntt, tgt, rng)
    return KeySet(context=ctx, secret_small=s.astype(np.int8), pk_ntt=pk_ntt, relin=relin,
                  galois=galois, s_ntt=s_ntt)


# ---------------------------------------------------------------------------
# ciphertexts
# ---------------------------------------------------------------------------
class FvCiphertext:
    """RNS ciphertext, resident in HBM as a (parts, k, N) uint32 tensor.

    ``parts`` reads as the reference's list of (k, N) int64 stacks
    (fv.py:30-42); assigning host parts uploads lazily."""

    __slots__ = ("_dev", "_host", "level_used", "params", "_live")

    def __init__(self, parts, level_used, params, dev=None):
        self._dev = dev
        self._host = None if parts is None else [np.asarray(p, dtype=np.int64) for p in parts]
        self.level_used = level_used
        self.params = params
        self._live = True

    @property
    def parts(self):
        if self._host is None:
            host = nat.to_host(self._dev).astype(np.int64)
            self._host = [host[i] for i in range(host.shape[0])]
        return self._host

    @parts.setter
    def parts(self, value):
        self._host = [np.asarray(p, dtype=np.int64) for p in value]
        self._dev = None

    def device(self):
        """The (parts, k, N) device stack.  Host parts (assigned, or read from
        a wire record) are uploaded by ``FvBackend.dev``, which validates
        them against the context first."""
        if self._dev is None:
            raise ParamMismatchError("host-side ciphertext parts: upload through FvBackend.dev(ct)")
        return self._dev

    @property
    def nparts(self) -> int:
        return self._dev.shape[0] if self._dev is not None else len(self._host)

    def __repr__(self):
        return f"FvCiphertext(parts={self.nparts}, level={self.level_used})"


# ---------------------------------------------------------------------------
# backend
# ---------------------------------------------------------------------------
class FvBackend(SlotBackend):
    """GPU implementation of the slot contract (fv.py:254-432)."""

    # layer_eval dispatches to the batched planner for this backend
    batched_layers = True

    def __init__(self, params: BackendParams, keys: KeySet = None, rng=None):
        if params.slot_count != params.ring_dimension // 2:
            raise ParamMismatchError("FV backend requires slot_count = n/2")
        super().__init__(params)
        self.rng = rng if rng is not None else np.random.default_rng()
        if keys is None:
            keys = keygen(FvParams.from_backend(params), rng=self.rng)
        elif not isinstance(keys, KeySet):
            # the reference's host KeySet (keygen / serialize.read_keyset,
            # fv.py:220-228): uploaded once into the device layout
            fp = keys.context.fp
            ctx = FvContext(FvParams(n=fp.n, t=fp.t, q_primes=list(fp.q_primes), sigma=fp.sigma))
            keys = KeySet.from_host(ctx, keys.secret, keys.public,
                                    (keys.relin.body, keys.relin.mask),
                                    {off: (sk.body, sk.mask) for off, sk in keys.galois.items()})
        self.keys = keys
        self.ctx = keys.context
        if self.ctx.t != params.plain_modulus or self.ctx.n != params.ring_dimension:
            raise ParamMismatchError("key set was generated for different parameters")
        ctx = self.ctx
        self._s_mont = ctx.to_mont(keys.s_ntt)
        self._s2_mont = ctx.to_mont(ctx.elementwise(2, keys.s_ntt, keys.s_ntt))
        self._pk_mont = ctx.to_mont(keys.pk_ntt.contiguous())
        self._e0_ntt = None

    # ---- device residency -------------------------------------------------------
    def dev(self, ct):
        """Device stack of any ciphertext with the reference's shape: this
        backend's handles directly; host parts (an ``FvCiphertext`` whose
        parts were assigned, or the reference's own ``FvCiphertext`` as
        ``serialize.read_ciphertext`` returns it, fv.py:30-42) are checked --
        2 or 3 components of shape (k, N), every residue in [0, p_j) -- and
        uploaded (cached on this backend's handles)."""
        if isinstance(ct, FvCiphertext) and ct._dev is not None:
            return ct._dev
        parts = ct._host if isinstance(ct, FvCiphertext) else ct.parts
        d = nat.to_device(self.check_host_parts(parts).astype(np.int32))
        if isinstance(ct, FvCiphertext):
            ct._dev = d
        return d

    def check_host_parts(self, parts) -> np.ndarray:
        ctx = self.ctx
        if len(parts) not in (2, 3):
            raise FormatError(f"FV ciphertext needs 2 or 3 components, got {len(parts)}")
        stack = []
        for comp in parts:
            arr = np.asarray(comp)
            if arr.shape != (ctx.k, ctx.n):
                raise FormatError(f"component shape {arr.shape} != ({ctx.k}, {ctx.n})")
            arr = arr.astype(np.int64)
            if (arr < 0).any() or (arr >= ctx.pcol).any():
                raise FormatError("residue outside [0, p_j)")
            stack.append(arr)
        return np.stack(stack)

    # ---- batching ----------------------------------------------------------
    def _slots_dev(self, vecs):
        torch = _torch()
        arr = np.asarray(vecs)
        arr = np.array(arr.tolist(), dtype=np.uint64) if arr.dtype == object else arr.astype(np.uint64)
        arr = arr.reshape(-1, self.ctx.n // 2)
        return nat.to_device(arr.view(np.int64))

    def _encode_dev(self, vecs):
        """(B, N/2) slot vectors -> (B, N) plaintext polys mod t (device)."""
        sl = self._slots_dev(vecs)
        out = self.ctx.empty(sl.shape[0], self.ctx.n, dtype=_torch().int64)
        self.ctx.call("hefv_encode", sl.data_ptr(), out.data_ptr(), sl.shape[0], self.ctx.stream())
        return out

    def _decode_dev(self, polys):
        out = self.ctx.empty(polys.shape[0], self.ctx.n // 2, dtype=_torch().int64)
        self.ctx.call("hefv_decode", polys.data_ptr(), out.data_ptr(), polys.shape[0],
                      self.ctx.stream())
        return out

    def _host_plain(self, dev) -> np.ndarray:
        arr = nat.to_host(dev)
        return arr if self.ctx.t < (1 << 31) else arr.astype(object)

    def encode(self, vec) -> np.ndarray:
        """Slot vector -> plaintext polynomial mod t (fv.py:280-285)."""
        t = self.ctx.t
        v = np.asarray(vec, dtype=object) % t if np.asarray(vec).dtype == object else \
            np.mod(np.asarray(vec, dtype=np.int64), t)
        return self._host_plain(self._encode_dev(v)[0])

    def decode(self, poly) -> np.ndarray:
        t = self.ctx.t
        p = np.asarray(poly)
        p = np.array([int(x) % t for x in p], dtype=np.uint64) if p.dtype == object else \
            np.mod(p.astype(np.int64), t).astype(np.uint64)
        dev = nat.to_device(p.view(np.int64).reshape(1, -1))
        return self._host_plain(self._decode_dev(dev)[0])

    def _rns_plain(self, polys, mode, to_ntt, montgomery):
        out = self.ctx.empty(polys.shape[0], self.ctx.k, self.ctx.n)
        self.ctx.call("hefv_plain_to_rns", polys.data_ptr(), out.data_ptr(), polys.shape[0],
                      mode, 1 if to_ntt else 0, 1 if montgomery else 0, self.ctx.stream())
        return out

    def _delta_m_dev(self, vec):
        return self._rns_plain(self._encode_dev(vec), 0, False, False)

    def _cmult_plain_dev(self, vec):
        return self._rns_plain(self._encode_dev(vec), 1, True, True)

    # ---- primitives -----------------------------------------------------------
    def _fresh(self, dev, level):
        return FvCiphertext(None, level, self.params, dev=dev)

    def _encrypt(self, vec):
        return self._encrypt_many(np.asarray(vec)[None])[0]

    def encrypt_many(self, values_list) -> list:
        """``[encrypt(v) for v in values_list]`` with one launch per stage; the
        Generator and the ledger see exactly the per-call sequence."""
        plains = [self.as_plain(v) for v in values_list]
        if not plains:
            return []
        cts = self._encrypt_many(plains)
        for _ in cts:
            self._c.bump("encrypt", level=0)
        return cts

    def _encrypt_many(self, vecs):
        """Encrypt B slot vectors; the Generator is consumed per ciphertext in
        the reference's order (u, e1, e2)."""
        torch = _torch()
        ctx = self.ctx
        B = len(vecs)
        u = np.empty((B, ctx.n), np.int8)
        e1 = np.empty((B, ctx.n), np.int8)
        e2 = np.empty((B, ctx.n), np.int8)
        for b in range(B):
            u[b] = ctx.rand_ternary(self.rng)
            e1[b] = ctx.rand_error(self.rng)
            e2[b] = ctx.rand_error(self.rng)
        slots = self._slots_dev(np.stack([np.asarray(v) for v in vecs]))
        out = ctx.empty(B, 2, ctx.k, ctx.n)
        ud, e1d, e2d = (nat.to_device(x) for x in (u, e1, e2))
        ctx.call("hefv_encrypt_slots", self._pk_mont.data_ptr(), ud.data_ptr(), e1d.data_ptr(),
                 e2d.data_ptr(), slots.data_ptr(), out.data_ptr(), B, ctx.stream())
        return [self._fresh(out[b], 0) for b in range(B)]

    def _decrypt_poly_dev(self, devs):
        ctx = self.ctx
        torch = _torch()
        nparts = devs[0].shape[0]
        cts = torch.stack(devs) if len(devs) > 1 else devs[0][None]
        B = cts.shape[0]
        out = ctx.empty(B, ctx.n, dtype=torch.int64)
        scratch = ctx.empty(B, ctx.k, ctx.n)
        ctx.call("hefv_decrypt", cts.data_ptr(), nparts, self._s_mont.data_ptr(),
                 self._s2_mont.data_ptr(), out.data_ptr(), scratch.data_ptr(), B, ctx.stream())
        return out

    def decrypt_poly(self, ct: FvCiphertext) -> np.ndarray:
        """Plaintext polynomial mod t (fv.py:337-349)."""
        return self._host_plain(self._decrypt_poly_dev([self.dev(ct)])[0])

    def _decrypt_slots_dev(self, devs):
        ctx = self.ctx
        torch = _torch()
        nparts = devs[0].shape[0]
        cts = torch.stack(devs) if len(devs) > 1 else devs[0][None]
        out = ctx.empty(cts.shape[0], ctx.n // 2, dtype=torch.int64)
        ctx.call("hefv_decrypt_slots", cts.data_ptr(), nparts, self._s_mont.data_ptr(),
                 self._s2_mont.data_ptr(), out.data_ptr(), cts.shape[0], ctx.stream())
        return out

    def _decrypt(self, ct):
        slots = self._decrypt_slots_dev([self.dev(ct)])[0]
        return np.asarray(self._host_plain(slots), dtype=self._dtype)

    def decrypt_slots_async(self, cts):
        """Queue the decryption of ``cts`` (same part count) and an
        asynchronous copy of the slots to pinned host memory; returns a
        callable that waits for that copy only (not for later launches) and
        gives the slot vectors.  Lets a stream of images decrypt image i
        while image i+1 is already queued."""
        torch = _torch()
        for ct in cts:
            self._check_params(ct)
        dev = self._decrypt_slots_dev([self.dev(ct) for ct in cts])
        host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
        host.copy_(dev, non_blocking=True)
        nat.TRAFFIC["d2h"] += host.numel() * host.element_size()
        done = torch.cuda.Event()
        done.record()

        def wait():
            done.synchronize()
            arr = host.numpy()
            return [np.asarray(arr[i] if self.ctx.t < (1 << 31) else arr[i].astype(object),
                               dtype=self._dtype) for i in range(arr.shape[0])]

        return wait

    def decrypt_many(self, cts) -> list:
        """Batched decryption of several ciphertexts (one launch per stage)."""
        if not cts:
            return []
        for ct in cts:
            self._check_params(ct)
        groups = {}
        for i, ct in enumerate(cts):
            groups.setdefault(ct.nparts, []).append(i)
        res = [None] * len(cts)
        for _, idx in groups.items():
            slots = self._decrypt_slots_dev([self.dev(cts[i]) for i in idx])
            host = nat.to_host(slots)
            for r, i in enumerate(idx):
                res[i] = np.asarray(host[r] if self.ctx.t < (1 << 31) else host[r].astype(object),
                                    dtype=self._dtype)
        return res

    # The primitives below are single calls of the object-level C-ABI
    # (api.cu): the Python side only allocates the output and passes pointers.
    def _add(self, a, b, level):
        da, db = self.dev(a), self.dev(b)
        m = min(da.shape[0], db.shape[0])
        da, db = da[:m].contiguous(), db[:m].contiguous()
        out = _torch().empty_like(da)
        self.ctx.call("hefv_add", da.data_ptr(), db.data_ptr(), m, out.data_ptr(),
                      self.ctx.stream())
        return self._fresh(out, level)

    def _add_plain(self, a, vec, level):
        slots = self._slots_dev(np.asarray(vec)[None])
        da = self.dev(a).contiguous()
        out = _torch().empty_like(da)
        self.ctx.call("hefv_add_plain", da.data_ptr(), da.shape[0], slots.data_ptr(),
                      out.data_ptr(), self.ctx.stream())
        return self._fresh(out, level)

    def _cmult(self, a, vec, level):
        slots = self._slots_dev(np.asarray(vec)[None])
        da = self.dev(a).contiguous()
        out = _torch().empty_like(da)
        self.ctx.call("hefv_cmult", da.data_ptr(), da.shape[0], slots.data_ptr(), out.data_ptr(),
                      self.ctx.stream())
        return self._fresh(out, level)

    def _mult(self, a, b, level):
        ctx = self.ctx
        da = self.dev(a)[:2].contiguous()
        db = da if b is a else self.dev(b)[:2].contiguous()
        out = ctx.empty(2, ctx.k, ctx.n)
        ctx.call("hefv_mult", da.data_ptr(), db.data_ptr(), self.keys.relin.handle,
                 out.data_ptr(), ctx.stream())
        return self._fresh(out, level)

    def _square_many_dev(self, devs, chunk=512):
        """Squares of B ciphertexts (device stacks), batched: one tensor launch
        sequence and one relinearisation key switch per chunk; each result is
        limb-identical to ``_mult(a, a)``.  Returns a list of (2, k, N)."""
        from .planner import keyswitch_call

        torch = _torch()
        ctx = self.ctx
        key = self.keys.relin
        stack = ctx.k * ctx.n
        res = []
        for lo in range(0, len(devs), chunk):
            part = devs[lo:lo + chunk]
            B = len(part)
            a = torch.stack([d[:2] for d in part]).contiguous()
            out3 = ctx.empty(B, 3, ctx.k, ctx.n)
            scratch = ctx.empty(B * 7 * ctx.a * ctx.n)
            ctx.call("hefv_mult_tensor_many", a.data_ptr(), 2 * stack, a.data_ptr(), 2 * stack,
                     out3.data_ptr(), scratch.data_ptr(), B, ctx.stream())
            del scratch, a
            out = ctx.empty(B, 2, ctx.k, ctx.n)
            keyswitch_call(ctx, key, out3[0, 2].data_ptr(), 3 * stack, out[0, 0].data_ptr(),
                           out[0, 1].data_ptr(), 2 * stack, None, out3[0, 0].data_ptr(),
                           out3[0, 1].data_ptr(), 3 * stack, None, None, 0, B)
            res += [out[i] for i in range(B)]
        return res

    def rotation_hops(self, offset: int) -> list:
        """Key-switch hops of a rotation (fv.py:422-425)."""
        if offset == 0:
            return []
        if offset in self.keys.galois:
            return [offset]
        return [1 << j for j in range(offset.bit_length()) if offset >> j & 1]

    def _hop(self, dev, off):
        ctx = self.ctx
        out = ctx.empty(2, ctx.k, ctx.n)
        ctx.call("hefv_rotate", dev.data_ptr(), galois_element(off, ctx.n),
                 self.keys.galois[off].handle, out.data_ptr(), ctx.stream())
        return out

    def _rotate(self, a, offset, level):
        dev = self.dev(a)
        if offset == 0:
            return self._fresh(dev.clone(), level)
        dev = dev[:2].contiguous()
        for off in self.rotation_hops(offset):
            dev = self._hop(dev, off)
        return self._fresh(dev, level)

    # ---- helpers for the layer planner ---------------------------------------------
    def layer_eval_batched(self, rows, x, skip_zero_segments=True, scale_factor=1):
        """A whole compiled layer through the batched planner: the limbs,
        levels, Generator draws and CostReport of the reference's per-row
        ``layer_eval`` (inference.py:261-349).  ``rows`` / ``x`` may be the
        reference's own ``WeightRow`` / ``PackedVector`` objects; the result
        has the type of ``x``."""
        from .errors import DimensionError
        from .planner import planned_layer_eval

        for row in rows:
            if row.length != x.logical_length:
                raise DimensionError(f"row length {row.length} != input length {x.logical_length}")
        res = planned_layer_eval(self, rows, x, skip_zero_segments, scale_factor)
        if type(res) is not type(x):
            res = type(x)(res.logical_length, res.slots_used, res.cts, scale=res.scale)
        return res

    def e0_plain_ntt(self):
        """Montgomery NTT of centred(encode(e0)), cached (inference.py:287, 327)."""
        if self._e0_ntt is None:
            self._e0_ntt = self._cmult_plain_dev(self.one_hot(0)[None])
        return self._e0_ntt


# ---------------------------------------------------------------------------
# op-sequence runner and conformance check (fv.py:435-479)
# ---------------------------------------------------------------------------
def run_sequence(backend: SlotBackend, ops) -> list:
    """Execute a declarative op list; returns the value stack."""
    stack = []
    for op in ops:
        kind = op[0]
        if kind == "enc":
            stack.append(backend.encrypt(op[1]))
        elif kind == "add":
            stack.append(backend.add(stack[op[1]], stack[op[2]]))
        elif kind == "mult":
            stack.append(backend.mult(stack[op[1]], stack[op[2]]))
        elif kind == "cmult":
            stack.append(backend.cmult(stack[op[1]], op[2]))
        elif kind == "add_plain":
            stack.append(backend.add_plain(stack[op[1]], op[2]))
        elif kind == "rotate":
            stack.append(backend.rotate(stack[op[1]], op[2]))
        elif kind == "psum":
            stack.append(backend.partial_sum(stack[op[1]], op[2]))
        elif kind == "asum":
            stack.append(backend.all_sum(stack[op[1]], op[2]))
        else:
            raise ValueError(f"unknown op {kind!r}")
    return stack


def fv_conformance(fv_backend, sim_backend, ops) -> bool:
    """Run ``ops`` on both backends; False on the first decryption mismatch."""
    fv_stack = run_sequence(fv_backend, ops)
    sim_stack = run_sequence(sim_backend, ops)
    for f, s in zip(fv_stack, sim_stack):
        got = np.asarray(fv_backend.decrypt(f), dtype=np.int64)
        want = np.asarray(sim_backend.decrypt(s), dtype=np.int64)
        if not np.array_equal(got, want):
            return False
    return True
