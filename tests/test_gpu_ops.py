"""GPU parity: every FV primitive bit-identical to the CPU oracle.

The oracle (oracle/fv_oracle.py) is pinned to the reference by
tests/test_oracle.py; here the CUDA path (through the C-ABI) must produce
the same ciphertext limbs under the same seeded keys and randomness.
"""

import json

import numpy as np
import pytest

from oracle import fv_oracle as O
from paper_1901_10074_b200.params import BackendParams, profile

pytestmark = pytest.mark.gpu


def _digest(parts):
    return O.limb_digest(parts)


# ---------------------------------------------------------------- NTT
@pytest.mark.parametrize("n,bits", [(16, 30), (64, 30), (1024, 30), (4096, 30), (16384, 30),
                                    (32768, 30), (64, 20), (4096, 50), (16384, 60),
                                    (32768, 55), (65536, 60)])
def test_ntt_matches_oracle(n, bits, rng):
    from paper_1901_10074_b200.ntt import NttPrime

    p = O.ntt_primes(1, bits, 2 * n)[0]
    ref = O.OracleNtt(p, n)
    gpu = NttPrime(p, n)
    assert gpu.psi == ref.psi
    a = np.array([int(rng.integers(0, p)) for _ in range(3 * n)], dtype=object).reshape(3, n)
    want = ref.fwd(a)
    got = gpu.fwd(a)
    assert np.array_equal(np.asarray(got, dtype=object), np.asarray(want, dtype=object))
    back = gpu.inv(got)
    assert np.array_equal(np.asarray(back, dtype=object), np.asarray(a % p, dtype=object))


def test_ntt_negacyclic_against_schoolbook(rng):
    from paper_1901_10074_b200.ntt import NttPrime

    n = 64
    p = O.ntt_primes(1, 30, 2 * n)[0]
    tr = NttPrime(p, n)
    a = rng.integers(0, p, n)
    b = rng.integers(0, p, n)
    want = O.schoolbook(a, b, n, p).astype(np.int64)
    assert np.array_equal(tr.negacyclic_mul(a, b), want)


# ---------------------------------------------------------------- FV desk
@pytest.fixture(scope="module")
def desk_pair():
    from paper_1901_10074_b200.fv import FvBackend

    p = profile("desk")
    gpu = FvBackend(p, rng=np.random.default_rng(77))
    orc = O.OracleFvBackend(p, rng=np.random.default_rng(77))
    return gpu, orc


def test_keys_match_oracle(desk_pair):
    gpu, orc = desk_pair
    assert np.array_equal(gpu.keys.secret, orc.keys.secret)
    for j in (0, 3, 5):
        assert np.array_equal(gpu.keys.relin.body[j], orc.keys.relin.body[j])
        assert np.array_equal(gpu.keys.relin.mask[j], orc.keys.relin.mask[j])
    assert sorted(gpu.keys.galois) == sorted(orc.keys.galois)
    for off in (1, 64, 1024):
        assert np.array_equal(gpu.keys.galois[off].body[2], orc.keys.galois[off].body[2])
    assert np.array_equal(gpu.keys.public[0], orc.keys.public[0])
    assert np.array_equal(gpu.keys.public[1], orc.keys.public[1])


def test_encode_decode_match(desk_pair, rng):
    gpu, orc = desk_pair
    t = gpu.params.plain_modulus
    v = rng.integers(0, t, gpu.params.slot_count)
    assert np.array_equal(gpu.encode(v), orc.encode(v))
    assert np.array_equal(gpu.decode(gpu.encode(v)), v % t)


def test_ops_bit_identical(desk_pair, rng):
    gpu, orc = desk_pair
    t = gpu.params.plain_modulus
    v = rng.integers(0, t, gpu.params.slot_count)
    w = rng.integers(0, t, gpu.params.slot_count)
    ga, oa = gpu.encrypt(v), orc.encrypt(v)
    assert _digest(ga.parts) == _digest(oa.parts)
    gb, ob = gpu.encrypt(w), orc.encrypt(w)
    cases = {
        "add": (gpu.add(ga, gb), orc.add(oa, ob)),
        "add_plain": (gpu.add_plain(ga, w), orc.add_plain(oa, w)),
        "cmult": (gpu.cmult(ga, w), orc.cmult(oa, w)),
        "rotate1": (gpu.rotate(ga, 1), orc.rotate(oa, 1)),
        "rotate129": (gpu.rotate(ga, 129), orc.rotate(oa, 129)),
        "rotate-17": (gpu.rotate(ga, -17), orc.rotate(oa, -17)),
        "mult": (gpu.mult(ga, gb), orc.mult(oa, ob)),
        "square": (gpu.mult(ga, ga), orc.mult(oa, oa)),
    }
    for name, (g, o) in cases.items():
        assert g.level_used == o.level_used, name
        assert _digest(g.parts) == _digest(o.parts), name
        assert np.array_equal(gpu.decrypt(g), orc.decrypt(o)), name


def test_decrypt_poly_and_three_parts(desk_pair, rng):
    gpu, orc = desk_pair
    t = gpu.params.plain_modulus
    v = rng.integers(0, t, gpu.params.slot_count)
    ga, oa = gpu.encrypt(v), orc.encrypt(v)
    assert np.array_equal(np.asarray(gpu.decrypt_poly(ga), dtype=np.int64),
                          np.asarray(orc.decrypt_poly(oa), dtype=np.int64))
    # unrelinearised 3-part ciphertext decrypts with s^2
    t3 = orc.tensor(oa, oa)
    from paper_1901_10074_b200.fv import FvCiphertext

    g3 = FvCiphertext(t3, 1, gpu.params)
    o3 = O.OracleCiphertext(t3, 1, orc.params)
    assert np.array_equal(np.asarray(gpu.decrypt_poly(g3), dtype=np.int64),
                          np.asarray(orc.decrypt_poly(o3), dtype=np.int64))


def test_folds_and_levels(desk_pair, rng):
    gpu, orc = desk_pair
    t = gpu.params.plain_modulus
    v = rng.integers(0, t, gpu.params.slot_count)
    ga, oa = gpu.encrypt(v), orc.encrypt(v)
    g = gpu.all_sum(gpu.cmult(ga, [1] * 100), 100)
    o = orc.all_sum(orc.cmult(oa, [1] * 100), 100)
    assert _digest(g.parts) == _digest(o.parts)
    g = gpu.partial_sum(ga, 8)
    o = orc.partial_sum(oa, 8)
    assert _digest(g.parts) == _digest(o.parts)


def test_host_parts_roundtrip(desk_pair, rng):
    from paper_1901_10074_b200.fv import FvCiphertext

    gpu, orc = desk_pair
    t = gpu.params.plain_modulus
    v = rng.integers(0, t, gpu.params.slot_count)
    oa = orc.encrypt(v)
    ga = FvCiphertext([p.copy() for p in oa.parts], 0, gpu.params)
    assert np.array_equal(gpu.decrypt(ga), v % t)
    g = gpu.rotate(ga, 5)
    o = orc.rotate(oa, 5)
    assert _digest(g.parts) == _digest(o.parts)


# ---------------------------------------------------------------- small custom params
def test_tiny_params_all_ops(rng):
    from paper_1901_10074_b200.fv import FvBackend

    p = BackendParams(ring_dimension=64, coeff_modulus_bits=120, plain_modulus=257,
                      slot_count=32, depth_budget=4)
    gpu = FvBackend(p, rng=np.random.default_rng(5))
    orc = O.OracleFvBackend(p, rng=np.random.default_rng(5))
    v = rng.integers(0, 257, 32)
    ga, oa = gpu.encrypt(v), orc.encrypt(v)
    assert _digest(ga.parts) == _digest(oa.parts)
    for g, o in [(gpu.mult(ga, ga), orc.mult(oa, oa)), (gpu.rotate(ga, 7), orc.rotate(oa, 7)),
                 (gpu.cmult(ga, v), orc.cmult(oa, v))]:
        assert _digest(g.parts) == _digest(o.parts)


@pytest.mark.parametrize("n,bits,seed", [(512, 120, 1), (1024, 240, 2), (1024, 270, 3),
                                         (2048, 330, 4), (2048, 600, 5)])
def test_random_op_sequences_match_oracle(n, bits, seed):
    """Seeded random op sequences (encrypt, add, add_plain, cmult, rotations by
    random offsets, squares and products, all_sum) over parameter sets that
    cross the per-prime / aux-basis key-switch boundary (k = 8 | 9..20):
    every intermediate ciphertext's limbs and level equal the oracle's."""
    from paper_1901_10074_b200.fv import FvBackend

    t = 12289  # = 1 mod 2N for every N here
    p = BackendParams(ring_dimension=n, coeff_modulus_bits=bits, plain_modulus=t,
                      slot_count=n // 2, depth_budget=6)
    gpu = FvBackend(p, rng=np.random.default_rng(seed))
    orc = O.OracleFvBackend(p, rng=np.random.default_rng(seed))
    g = np.random.default_rng(100 + seed)
    vecs = [g.integers(0, t, n // 2) for _ in range(3)]
    gs = [gpu.encrypt(v) for v in vecs]
    os_ = [orc.encrypt(v) for v in vecs]
    for step in range(10):
        op = g.integers(0, 6)
        i, j = (int(x) for x in g.integers(0, len(gs), 2))
        w = g.integers(0, t, n // 2)
        if op == 0:
            a, b = gpu.add(gs[i], gs[j]), orc.add(os_[i], os_[j])
        elif op == 1:
            a, b = gpu.add_plain(gs[i], w), orc.add_plain(os_[i], w)
        elif op == 2:
            a, b = gpu.cmult(gs[i], w % 17), orc.cmult(os_[i], w % 17)
        elif op == 3:
            off = int(g.integers(-n // 2 + 1, n // 2))
            a, b = gpu.rotate(gs[i], off), orc.rotate(os_[i], off)
        elif op == 4 and max(gs[i].level_used, gs[j].level_used) < 3:
            a, b = gpu.mult(gs[i], gs[j]), orc.mult(os_[i], os_[j])
        else:
            a, b = gpu.all_sum(gs[i], 8), orc.all_sum(os_[i], 8)
        assert a.level_used == b.level_used, (step, op)
        assert _digest(a.parts) == _digest(b.parts), (step, op)
        gs.append(a)
        os_.append(b)
    assert np.array_equal(gpu.decrypt(gs[-1]), orc.decrypt(os_[-1]))


def test_desk_golden_replay_matches_reference():
    """The reference's own desk run (seed 77, 10 ops) replayed on the GPU."""
    import json
    from pathlib import Path

    from paper_1901_10074_b200.fv import FvBackend
    from goldens import replay_ops

    g = json.loads((Path(__file__).resolve().parent / "golden" / "fv_desk.json").read_text())
    be = FvBackend(profile("desk"), rng=np.random.default_rng(g["seed"]))
    k = be.keys
    assert O.limb_digest([k.secret]) == g["secret"]
    assert O.limb_digest(list(k.public)) == g["pk"]
    assert O.limb_digest(list(k.relin.body) + list(k.relin.mask)) == g["relin"]
    for off, d in g["galois"].items():
        sk = k.galois[int(off)]
        assert O.limb_digest(list(sk.body) + list(sk.mask)) == d, off
    got, want = replay_ops(be, g)
    for key, val in got.items():
        assert val == want[key], key


def test_tiny_golden_full_limbs():
    import json
    from pathlib import Path

    from paper_1901_10074_b200.fv import FvBackend

    g = json.loads((Path(__file__).resolve().parent / "golden" / "fv_tiny.json").read_text())
    p = BackendParams(**g["params"])
    be = FvBackend(p, rng=np.random.default_rng(g["key_seed"]))
    v = np.random.default_rng(g["data_seed"]).integers(0, 257, 32)
    a = be.encrypt(v)
    assert [x.tolist() for x in a.parts] == g["enc"]
    assert [x.tolist() for x in be.mult(a, a).parts] == g["square"]
    assert [x.tolist() for x in be.rotate(a, 7).parts] == g["rotate7"]
    assert [x.tolist() for x in be.cmult(a, v).parts] == g["cmult"]


@pytest.mark.parametrize("case", json.loads((__import__("pathlib").Path(__file__).resolve().parent
                                             / "golden" / "ntt.json").read_text())["cases"],
                         ids=lambda c: f"n{c['n']}b{c['bits']}")
def test_ntt_golden_vectors(case):
    from paper_1901_10074_b200.ntt import NttPrime

    n, p = case["n"], case["p"]
    tr = NttPrime(p, n)
    assert tr.psi == case["psi"]
    rng = np.random.default_rng(case["seed"])
    a = np.array([int(rng.integers(0, p)) for _ in range(n)], dtype=object)
    fa = tr.fwd(a)
    assert O.limb_digest([np.asarray([int(x) for x in fa], dtype=np.int64)]) == case["fwd_digest"]
    assert [int(x) for x in tr.inv(fa)] == [int(x) for x in a]


# ---------------------------------------------------------------- race stress
@pytest.mark.parametrize("log_n,bits", [(10, 30), (12, 30), (13, 30), (14, 30), (15, 30),
                                        (16, 30), (10, 50), (12, 50), (13, 60), (14, 55),
                                        (15, 55), (16, 60)])
def test_transform_roundtrip_stress(log_n, bits):
    """Many CTAs, repeated: device-order forward then inverse must be the
    identity bit for bit (catches exchange/barrier races)."""
    import ctypes as C

    import torch

    from paper_1901_10074_b200 import _native as nat
    from paper_1901_10074_b200.ring import root_of_unity

    n = 1 << log_n
    primes = O.ntt_primes(4, bits, 2 * n)
    psis = [root_of_unity(p, n) for p in primes]
    lib = nat.load()
    h = C.c_void_p()
    wide = bits > 30
    if wide:
        nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 0, None, None, 4,
                                      (C.c_uint64 * 4)(*primes), (C.c_uint64 * 4)(*psis)))
        gen = torch.Generator(device="cuda").manual_seed(log_n)
        x = torch.randint(0, 1 << 40, (64, 4, n), dtype=torch.int64, device="cuda", generator=gen)
        x = x % torch.tensor(primes, dtype=torch.int64, device="cuda").view(1, 4, 1)
        fwd, inv = lib.hefv_ntt_fwd64, lib.hefv_ntt_inv64
    else:
        nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 4, (C.c_uint32 * 4)(*primes),
                                      (C.c_uint32 * 4)(*psis), 0, None, None))
        gen = torch.Generator(device="cuda").manual_seed(log_n)
        x = torch.randint(0, 1 << 29, (64, 4, n), dtype=torch.int32, device="cuda", generator=gen)
        fwd, inv = lib.hefv_ntt_fwd32, lib.hefv_ntt_inv32
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        nat.check(fwd(h, x.data_ptr(), y.data_ptr(), 64, 4, 0, 0, st))
        nat.check(inv(h, y.data_ptr(), z.data_ptr(), 64, 4, 0, 0, st))
        assert torch.equal(z, x)
    lib.hefv_ctx_destroy(h)


@pytest.mark.parametrize("log_n,bits", [(10, 50), (12, 50), (13, 60), (14, 60), (12, 20),
                                        (15, 55), (16, 60)])
def test_ntt64_device_order_matches_oracle(log_n, bits):
    """Batched 64-bit device-order transforms (the persistent k_ntt64_b path,
    several primes per CTA range, inputs up to 2^64 - 1) equal the oracle's
    natural-order NTT of x mod p permuted into bit-reversed order, and the
    inverse maps them back to x mod p."""
    import ctypes as C

    import torch

    from paper_1901_10074_b200 import _native as nat
    from paper_1901_10074_b200.ring import root_of_unity

    n = 1 << log_n
    L, B = (3, 5) if log_n <= 14 else (2, 3)
    primes = O.ntt_primes(L, bits, 2 * n)
    psis = [root_of_unity(p, n) for p in primes]
    lib = nat.load()
    h = C.c_void_p()
    nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 0, None, None, L,
                                  (C.c_uint64 * L)(*primes), (C.c_uint64 * L)(*psis)))
    g = np.random.default_rng(log_n * 100 + bits)
    xs = g.integers(0, 1 << 63, (B, L, n), dtype=np.uint64) * np.uint64(2) + g.integers(
        0, 2, (B, L, n), dtype=np.uint64)
    xs[0, 0, :4] = [0, 2**64 - 1, primes[0], primes[0] - 1]
    x = torch.from_numpy(xs.view(np.int64)).cuda()
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    nat.check(lib.hefv_ntt_fwd64(h, x.data_ptr(), y.data_ptr(), B, L, 0, 0, st))
    nat.check(lib.hefv_ntt_inv64(h, y.data_ptr(), z.data_ptr(), B, L, 0, 0, st))
    got = y.cpu().numpy().view(np.uint64)
    back = z.cpu().numpy().view(np.uint64)
    rev = np.array([int(format(i, f"0{log_n}b")[::-1], 2) for i in range(n)])
    for j, p in enumerate(primes):
        ref = O.OracleNtt(p, n)
        for b in (0, B - 1):
            red = np.array([int(v) % p for v in xs[b, j]], dtype=object)
            want = np.asarray(ref.fwd(red), dtype=object)[rev]
            assert np.array_equal(got[b, j].astype(object), want), (b, j)
            assert np.array_equal(back[b, j].astype(object), red), (b, j)
    lib.hefv_ctx_destroy(h)


@pytest.mark.parametrize("log_n,bits", [(10, 30), (12, 30), (13, 30), (14, 30), (15, 30),
                                        (16, 30), (14, 28), (12, 24)])
def test_ntt32_device_order_matches_oracle(log_n, bits):
    """Batched 30-bit device-order transforms (the persistent k_ntt32_b, the
    32-word single CTA at 2^15 and the split outer-pass + sub-transform form at
    2^16; prime boundaries inside CTA ranges, inputs up to 2^32 - 1)
    equal the oracle's natural-order NTT permuted into bit-reversed order,
    and invert to x mod p."""
    import ctypes as C

    import torch

    from paper_1901_10074_b200 import _native as nat
    from paper_1901_10074_b200.ring import root_of_unity

    n = 1 << log_n
    L, B = (3, 7) if log_n <= 14 else (2, 3)
    primes = O.ntt_primes(L, bits, 2 * n)  # 28/24-bit: the Barrett input path
    psis = [root_of_unity(p, n) for p in primes]
    lib = nat.load()
    h = C.c_void_p()
    nat.check(lib.hefv_ctx_create(C.byref(h), log_n, L, (C.c_uint32 * L)(*primes),
                                  (C.c_uint32 * L)(*psis), 0, None, None))
    g = np.random.default_rng(log_n)
    xs = g.integers(0, 1 << 32, (B, L, n), dtype=np.uint64).astype(np.uint32)
    x = torch.from_numpy(xs.view(np.int32)).cuda()
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    nat.check(lib.hefv_ntt_fwd32(h, x.data_ptr(), y.data_ptr(), B, L, 0, 0, st))
    nat.check(lib.hefv_ntt_inv32(h, y.data_ptr(), z.data_ptr(), B, L, 0, 0, st))
    got = y.cpu().numpy().view(np.uint32)
    back = z.cpu().numpy().view(np.uint32)
    rev = np.array([int(format(i, f"0{log_n}b")[::-1], 2) for i in range(n)])
    for j, p in enumerate(primes):
        ref = O.OracleNtt(p, n)
        for b in sorted({0, min(3, B - 1), B - 1}):
            red = xs[b, j].astype(np.int64) % p
            want = np.asarray(ref.fwd(red), dtype=np.int64)[rev]
            assert np.array_equal(got[b, j].astype(np.int64), want), (b, j)
            assert np.array_equal(back[b, j].astype(np.int64), red), (b, j)
    lib.hefv_ctx_destroy(h)


@pytest.mark.parametrize("name", ["desk", "retina"])
def test_mul_plain_and_keyswitch_batch_stress(name):
    import torch

    from paper_1901_10074_b200.fv import FvBackend
    from paper_1901_10074_b200.ring import galois_element

    p = profile(name)
    be = FvBackend(p, rng=np.random.default_rng(2))
    ctx = be.ctx
    k, n = ctx.k, ctx.n
    stack = k * n
    a = be.encrypt(np.arange(p.slot_count) % 11)
    # NTT-domain constant 1 in Montgomery form (2^32 mod q_j at every point)
    one = torch.tensor([[(1 << 32) % q] * n for q in ctx.q_primes], dtype=torch.int64)
    one = one.to(torch.int32).view(1, k, n).cuda()
    B = 64
    acc = torch.stack([a.device()] * B).contiguous()
    out = torch.empty_like(acc)
    for _ in range(3):
        ctx.call("hefv_mul_plain", acc.data_ptr(), one.data_ptr(), out.data_ptr(), B, 2, 1,
                 ctx.stream())
        assert torch.equal(out, acc)
    scr = torch.empty_like(acc)
    key = be.keys.galois[1]
    ctx.call("hefv_automorph", acc.data_ptr(), 2 * stack, None, scr.data_ptr(), 2,
             galois_element(1, n), B, ctx.stream())
    ctx.call("hefv_keyswitch", key.body_dev.data_ptr(), key.mask_dev.data_ptr(),
             scr.data_ptr() + stack * 4, 2 * stack, out.data_ptr(), out.data_ptr() + stack * 4,
             2 * stack, None, scr.data_ptr(), None, 2 * stack, None, None, 0, B, ctx.stream())
    single = be.rotate(a, 1).device()
    for b in range(B):
        assert torch.equal(out[b], single)


def test_custom_rotation_keys_single_hop():
    """keygen(rotation_offsets=...) adds non-power-of-two Galois keys; such a
    rotation is one hop (fv.py:422-425), bit-identical to the oracle."""
    from paper_1901_10074_b200.fv import FvBackend, FvParams, keygen

    p = profile("desk")
    fp = FvParams.from_backend(p)
    gk = keygen(fp, rotation_offsets={5, 100, -3}, rng=np.random.default_rng(8))
    assert {5, 100, 2045} <= set(gk.galois)
    gpu = FvBackend(p, keys=gk, rng=np.random.default_rng(9))
    ok = O.keygen(O.OracleParams.from_backend(p), rotation_offsets={5, 100, -3},
                  rng=np.random.default_rng(8))
    orc = O.OracleFvBackend(p, keys=ok, rng=np.random.default_rng(9))
    assert np.array_equal(gpu.keys.galois[100].body[1], orc.keys.galois[100].body[1])
    v = np.random.default_rng(1).integers(0, p.plain_modulus, p.slot_count)
    ga, oa = gpu.encrypt(v), orc.encrypt(v)
    for off in (5, 100, -3, 7):
        assert _digest(gpu.rotate(ga, off).parts) == _digest(orc.rotate(oa, off).parts), off
    assert gpu.rotation_hops(5) == [5] and gpu.rotation_hops(7) == [1, 2, 4]


def test_planner_with_custom_keys_and_empty_layer():
    from paper_1901_10074_b200 import inference as I
    from paper_1901_10074_b200.fv import FvBackend, FvParams, keygen

    p = profile("desk")
    s = p.slot_count
    results = []
    for planned in (True, False):
        gk = keygen(FvParams.from_backend(p), rotation_offsets={s - 3, s - 10},
                    rng=np.random.default_rng(3))
        be = FvBackend(p, keys=gk, rng=np.random.default_rng(4))
        x = I.pack_image(be, np.arange(300).reshape(1, 1, -1))
        rows = [I.WeightRow(out_index=i, length=300, slots_used=s,
                            positions=np.array([i, i + 1], dtype=np.int64),
                            values=np.array([2, -1], dtype=np.int64)) for i in range(12)]
        out = I.layer_eval(be, rows, x) if planned else I._serial_layer_eval(be, rows, x, True, 1)
        empty = I.layer_eval(be, [], x) if planned else I._serial_layer_eval(be, [], x, True, 1)
        results.append(([_digest(ct.parts) for ct in out.cts + empty.cts],
                        be.cost_report().as_dict(), I.decrypt_logits(be, out)))
    assert results[0][0] == results[1][0]
    assert results[0][1] == results[1][1]
    want = [2 * i - (i + 1) for i in range(12)]
    assert [int(v) for v in results[0][2]] == want
