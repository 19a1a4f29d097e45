"""Host-side logic (no GPU): C-ABI exports, prime/root precompute, the slot
contract + simulator, the planner's ledger replay and op counts."""

import json
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1901_10074_b200 import engine as E
from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200 import planner as PL
from paper_1901_10074_b200 import ring
from paper_1901_10074_b200.errors import DepthBudgetError, DimensionError, ParamMismatchError
from paper_1901_10074_b200.params import BackendParams, profile

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"


# ---------------------------------------------------------------- C-ABI
def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_1901_10074_b200 import _native

    header = (ROOT / "include" / "hefv.h").read_text()
    declared = set(re.findall(r"\b(hefv_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    path = _native.lib_path()
    assert path.exists(), "libhefv.so must be built (build())"
    lib = ctypes.CDLL(str(path))
    missing = [name for name in sorted(declared) if not hasattr(lib, name)]
    assert not missing, missing
    # the ctypes binding covers the header
    assert declared <= set(_native.EXPORTED) | {"hefv_ctx_destroy"}


def test_no_cpu_fallback_without_device(monkeypatch):
    from paper_1901_10074_b200 import _native
    from paper_1901_10074_b200.errors import NativeError

    monkeypatch.setattr(_native, "cuda_available", lambda: False)
    monkeypatch.delenv("HEFV_ALLOW_NO_CUDA", raising=False)
    with pytest.raises(NativeError):
        _native.require_device()


# ---------------------------------------------------------------- precompute
def test_primes_roots_match_reference():
    g = json.loads((GOLD / "primes.json").read_text())
    for name in ("desk", "mnist", "retina"):
        p = profile(name)
        count = max(2, -(-p.coeff_modulus_bits // ring.WORD_BITS))
        q = ring.find_ntt_primes(count, ring.WORD_BITS, 2 * p.ring_dimension)
        assert q == g[name]["q"]
        assert [ring.root_of_unity(x, p.ring_dimension) for x in q] == g[name]["q_psi"]
        assert ring.root_of_unity(p.plain_modulus, p.ring_dimension) == g[name]["t_psi"]
        qq = 1
        for x in q:
            qq *= x
        bits = p.ring_dimension.bit_length() + 2 * qq.bit_length() + 2
        aux = ring.find_ntt_primes(-(-bits // 29), 30, 2 * p.ring_dimension, below=min(q))
        assert aux == g[name]["aux"]
    p720 = profile("retina").replace(coeff_modulus_bits=720)
    assert ring.find_ntt_primes(24, 30, 2 * p720.ring_dimension) == g["retina-720"]["q"]


def test_crt_constants_and_words():
    primes = ring.find_ntt_primes(5, 30, 64)
    cc = ring.CrtConstants.build(primes)
    prod = 1
    for p in primes:
        prod *= p
    assert cc.product == prod
    back = sum(int(w) << (32 * i) for i, w in enumerate(cc.prod_words))
    assert back == prod
    for i, p in enumerate(primes):
        hat = sum(int(w) << (32 * k) for k, w in enumerate(cc.hat_words[i]))
        assert hat == prod // p and hat * int(cc.hat_inv[i]) % p == 1


def test_bitrev_and_slot_map():
    rev = ring.bitrev_perm(6)
    assert sorted(rev.tolist()) == list(range(64)) and rev[1] == 32
    s2e = ring.slot_to_eval(16)
    assert s2e[0] == 0 and s2e[1] == 1 and len(set(s2e.tolist())) == 8


# ---------------------------------------------------------------- contract + simulator
@pytest.fixture
def tiny():
    return E.SimBackend(BackendParams(ring_dimension=16, coeff_modulus_bits=120, plain_modulus=17,
                                      slot_count=8, depth_budget=3))


def test_sim_rotate_and_folds(tiny):
    v = np.arange(8)
    ct = tiny.encrypt(v)
    assert np.array_equal(tiny.decrypt(tiny.rotate(ct, 3)), np.roll(v, -3) % 17)
    assert np.array_equal(tiny.decrypt(tiny.rotate(ct, -1)), np.roll(v, 1) % 17)
    ps = tiny.decrypt(tiny.partial_sum(ct, 4))
    assert ps[0] == sum(range(4)) % 17 and ps[4] == sum(range(4, 8)) % 17
    ps3 = tiny.decrypt(tiny.partial_sum(ct, 3))
    assert ps3[0] == 3 and ps3[3] == 12
    assert tiny.decrypt(tiny.all_sum(tiny.encrypt([1, 2, 3]), 3))[0] == 6


def test_sim_errors_and_ledger(tiny):
    with pytest.raises(DimensionError):
        tiny.as_plain(np.zeros(9))
    with pytest.raises(DimensionError):
        tiny.as_plain(np.zeros((2, 2)))
    a = tiny.encrypt([1])
    b = tiny.cmult(tiny.cmult(tiny.cmult(a, [1]), [1]), [1])
    with pytest.raises(DepthBudgetError):
        tiny.cmult(b, [1])
    other = E.SimBackend(profile("desk"))
    with pytest.raises(ParamMismatchError):
        tiny.add(a, other.encrypt([1]))
    rep = tiny.cost_report()
    assert rep.cmult_count == 3 and rep.encrypt_count == 1 and rep.max_level_used == 3
    assert rep.peak_live_ciphertexts == 4
    tiny.release(a, a)
    assert tiny.cost_report().peak_live_ciphertexts == 4


def _random_rows(rng, length, s, count):
    rows = []
    for i in range(count):
        nnz = int(rng.integers(0, 10))
        pos = np.sort(rng.choice(length, size=nnz, replace=False)).astype(np.int64)
        vals = rng.integers(1, 9, nnz).astype(np.int64)
        rows.append(I.WeightRow(out_index=i, length=length, slots_used=s, positions=pos,
                                values=vals, bias=int(rng.integers(-3, 4)) if i % 4 == 0 else 0))
    return rows


@pytest.mark.parametrize("s,skip", [(8, True), (8, False), (5, True), (4, True)])
def test_ledger_replay_matches_serial_schedule(s, skip):
    """The planner's ledger replay equals the serial schedule's counters."""
    params = BackendParams(ring_dimension=16, coeff_modulus_bits=120, plain_modulus=17,
                           slot_count=8, depth_budget=4)
    rng = np.random.default_rng(s * 10 + skip)
    length = 3 * s - 1
    rows = _random_rows(rng, length, s, 23)
    data = rng.integers(0, 5, length)

    sim = E.SimBackend(params)
    x = I.pack_image(sim, data.reshape(1, 1, -1), slots_used=s)
    before = sim.cost_report()
    I._serial_layer_eval(sim, rows, x, skip, 1)
    want = sim.cost_report()

    sim2 = E.SimBackend(params)
    x2 = I.pack_image(sim2, data.reshape(1, 1, -1), slots_used=s)
    assert sim2.cost_report() == before
    R = len(rows)
    out_index = np.array([r.out_index for r in rows])
    seg_lists = [r.segment_ids if skip else np.arange(x2.k) for r in rows]
    nseg = np.array([len(sl) for sl in seg_lists])
    row_level = np.array([1 if n else 0 for n in nseg])
    seen, plain_bias = PL.replay_ledger(sim2._c, rows, x_k=x2.k, s=s, width=8,
                                        n_iter=PL._allsum_iters(s), m_arr=out_index // s,
                                        off_arr=out_index % s, bias_arr=[r.bias for r in rows],
                                        nseg=nseg, row_level=row_level)
    for m in range(max(1, -(-R // s))):
        if m not in seen:
            sim2.encrypt(plain_bias.get(m, np.zeros(8, dtype=np.int64)))
        elif m in plain_bias:
            sim2._c.bump("add", level=0)
    got = sim2.cost_report()
    assert got == want


def test_workload_op_counts_match_reference_config1():
    from paper_1901_10074_b200.configs import workload_op_counts

    g = json.loads((GOLD / "config1.json").read_text())
    c = workload_op_counts(1)
    for key in ("cmult", "add", "rotation", "encrypt", "mult"):
        assert c[key] == g["cost"][key], key
    assert c["ks_hops"] == 1873  # 1,872 hops + 1 relinearisation


def test_workload_op_counts_config2():
    from paper_1901_10074_b200.configs import workload_op_counts

    c = workload_op_counts(2)
    assert (c["cmult"], c["rotation"], c["ks_hops"], c["mult"]) == (21626, 148145, 208902, 2)


def test_simulator_config1_matches_plaintext_mod_t():
    from paper_1901_10074_b200.configs import (centred_mod, config_network, config_params,
                                               plaintext_forward)

    img, net = config_network(1)
    params = config_params(1)
    sim = E.SimBackend(params)
    logits = I.decrypt_logits(sim, I.infer(sim, net, I.pack_image(sim, img)))
    g = json.loads((GOLD / "config1.json").read_text())
    assert [int(v) for v in logits] == g["logits"]
    assert [int(v) for v in logits] == centred_mod(plaintext_forward(net, img),
                                                   params.plain_modulus)


def test_ks64_aux_prime_count_covers_the_exactness_bound():
    """rns.aux_prime_count: the aux basis of the 64-bit key switch must exceed
    8 L N max(p)^2 (ks64_aux.cu) for every config-4 shape; the setup rejects
    a basis that does not (checked on the GPU side as well)."""
    import math

    from paper_1901_10074_b200.ring import find_ntt_primes
    from paper_1901_10074_b200.rns import aux_prime_count

    for log_n in (10, 12, 14, 16):
        for L in (1, 2, 4, 8):
            for bits in (50, 60, 62):
                primes = find_ntt_primes(L, bits, 2 << log_n)
                T = aux_prime_count(primes, log_n)
                aux = find_ntt_primes(T, 30, 2 << log_n, below=int(2 ** 29.5))
                need = 3 + math.log2(L) + log_n + 2 * math.log2(max(primes))
                assert sum(math.log2(a) for a in aux) > need + 0.01
                assert max(aux) ** 2 * L < 2 ** 62  # MAC sums stay below 2^62
                assert T <= 6
