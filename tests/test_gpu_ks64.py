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
