"""Config 4: the RNS key switch over 50-62-bit primes, bit-exact against the
oracle's restatement of _keyswitch_apply (fv.py:205-217, object-dtype path)."""

import numpy as np
import pytest

from oracle import fv_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_ctx(primes, n):
    class Ctx:
        pass

    ctx = Ctx()
    ctx.n = n
    ctx.q_ntt = [O.OracleNtt(p, n) for p in primes]

    class FP:
        q_primes = primes

    ctx.fp = FP()
    return ctx


@pytest.mark.parametrize("path", ["direct", "aux"])
@pytest.mark.parametrize("n,L,bits", [(4096, 1, 50), (4096, 2, 60), (1024, 4, 55),
                                      (4096, 8, 50)])
def test_keyswitch64_matches_oracle(n, L, bits, path):
    from paper_1901_10074_b200.rns import RnsKeySwitch64

    primes = O.ntt_primes(L, bits, 2 * n)
    rng = np.random.default_rng(n + L)
    body = [np.array([[int(rng.integers(0, p)) for _ in range(n)] for _ in range(L)],
                     dtype=object) for p in primes]
    mask = [np.array([[int(rng.integers(0, p)) for _ in range(n)] for _ in range(L)],
                     dtype=object) for p in primes]
    c = np.array([[int(rng.integers(0, p)) for _ in range(n)] for p in primes], dtype=object)
    ctx = _oracle_ctx(primes, n)
    d0, d1 = O.keyswitch(ctx, c, O.OracleSwitchKey(body, mask))
    ks = RnsKeySwitch64(primes, n, aux=True)
    assert ks.aux
    key = ks.upload_key(body, mask)
    got = ks.switch_host(key, c[None], path)
    assert np.array_equal(got[0, 0].astype(object), np.asarray(d0, dtype=object))
    assert np.array_equal(got[0, 1].astype(object), np.asarray(d1, dtype=object))


@pytest.mark.parametrize("log_n,L,bits", [(10, 8, 62), (12, 8, 60), (13, 3, 50), (14, 8, 60),
                                          (15, 2, 55), (16, 8, 60), (16, 1, 61)])
def test_keyswitch64_aux_equals_direct(log_n, L, bits):
    """The aux-basis key switch (T ~29.5-bit primes, exact integer convolution
    reduced mod p_j) returns the direct 64-bit path's limbs for random and
    extreme digits / keys (all p - 1: the top of the exactness bound)."""
    import torch

    from paper_1901_10074_b200.rns import RnsKeySwitch64

    n = 1 << log_n
    primes = O.ntt_primes(L, bits, 2 * n)
    ks = RnsKeySwitch64(primes, n, aux=True)
    assert ks.aux
    p = torch.tensor(primes, dtype=torch.int64, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(log_n * 10 + L)
    B = 3
    dig = torch.randint(0, 1 << 62, (B, L, n), dtype=torch.int64, device="cuda",
                        generator=g) % p.view(1, L, 1)
    dig[1] = (p - 1).view(L, 1)                      # every digit p_i - 1
    dig[2, :, ::2] = 0
    dig[2, :, 1::2] = (p - 1).view(L, 1)
    for kind in ("random", "extreme"):
        if kind == "random":
            key = ks.random_key(log_n)
        else:
            top = (p - 1).view(L, 1, 1).expand(L, L, n).contiguous()
            key = ks._make_key(top, top.clone())
        a = ks.switch(key, dig, "aux")
        d = ks.switch(key, dig, "direct")
        assert torch.equal(a, d), kind


@pytest.mark.slow
def test_keyswitch64_large_n_matches_oracle():
    from paper_1901_10074_b200.rns import RnsKeySwitch64

    n, L = 32768, 2
    primes = O.ntt_primes(L, 55, 2 * n)
    rng = np.random.default_rng(7)
    mk = lambda p: np.array([int(v) for v in rng.integers(0, p, n, dtype=np.uint64)], dtype=object)  # noqa: E731
    body = [np.stack([mk(p) for _ in range(L)]) for p in primes]
    mask = [np.stack([mk(p) for _ in range(L)]) for p in primes]
    c = np.stack([mk(p) for p in primes])
    d0, d1 = O.keyswitch(_oracle_ctx(primes, n), c, O.OracleSwitchKey(body, mask))
    ks = RnsKeySwitch64(primes, n, aux=True)
    got = ks.switch_host(ks.upload_key(body, mask), c[None], "aux")
    assert np.array_equal(got[0, 0].astype(object), np.asarray(d0, dtype=object))
    assert np.array_equal(got[0, 1].astype(object), np.asarray(d1, dtype=object))


_KS64 = None


def _ks64_gold():
    global _KS64
    if _KS64 is None:
        import json
        from pathlib import Path

        _KS64 = json.loads((Path(__file__).resolve().parent / "golden" / "ks64.json")
                           .read_text())["cases"]
    return _KS64


@pytest.mark.parametrize("case", [pytest.param(i, marks=pytest.mark.slow) if i >= 5 else i
                                  for i in range(7)])
def test_keyswitch64_matches_reference_golden(case):
    """Config 4 pinned to the REFERENCE: _keyswitch_key + _keyswitch_apply
    (fv.py:176-217) over _FvContext(FvParams(N, t, 60-bit primes)) ran in
    tests/golden/make_golden.py --ks64 for (N, L) in {2^12, 2^14} x {2, 4, 8}
    and (2^16, 2).  The oracle regenerates the same key and input from the
    seed (their digests must equal the reference's), and both GPU paths
    (direct 64-bit and aux basis) must return the reference's d0 / d1."""
    from paper_1901_10074_b200.rns import RnsKeySwitch64

    g = _ks64_gold()[case]
    n, primes = g["n"], g["primes"]
    key, c = O.ks64_case(primes, n, g["seed"])
    assert O.limb_digest(list(key.body) + list(key.mask)) == g["key"]
    assert O.limb_digest([c]) == g["c"]
    ks = RnsKeySwitch64(primes, n, aux=True)
    dev_key = ks.upload_key(key.body, key.mask)
    for path in ("direct", "aux"):
        got = ks.switch_host(dev_key, c.astype(object)[None], path)
        assert O.limb_digest([got[0, 0].astype(np.int64)]) == g["d0"], path
        assert O.limb_digest([got[0, 1].astype(np.int64)]) == g["d1"], path
