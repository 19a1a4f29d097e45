"""The aux-basis key switch (ks_aux.cu) against the per-prime one
(ks_kernel.cu): both compute _keyswitch_apply (fv.py:205-217) and must give
identical limbs for any digits, key, epilogue addends and slot map -- the
aux path computes the integer convolution sum_i c_i (*) B_ji exactly in a
three-prime basis and reduces it mod p_j.

Digit limbs are drawn over the whole range [0, p_i) including the extremes
(0 and p_i - 1 runs), which maximise |sum| against the CRT bound."""

import numpy as np
import pytest

from paper_1901_10074_b200.params import BackendParams, profile
from paper_1901_10074_b200.ring import find_ntt_primes

pytestmark = pytest.mark.gpu


def _params(logn, k):
    n = 1 << logn
    t = find_ntt_primes(1, 40, 2 * n)[0]
    return BackendParams(ring_dimension=n, coeff_modulus_bits=30 * k, plain_modulus=t,
                         slot_count=n // 2, depth_budget=4)


def _both(params, B, seed, extremes=False):
    import torch

    from paper_1901_10074_b200.fv import FvBackend
    from paper_1901_10074_b200.ring import galois_element

    be = FvBackend(params, rng=np.random.default_rng(seed))
    ctx = be.ctx
    assert ctx.ks_aux, "aux key switch not enabled for this parameter set"
    k, n = ctx.k, ctx.n
    stack = k * n
    rng = np.random.default_rng(seed + 1)
    p = np.array(ctx.q_primes, dtype=np.int64)[None, :, None]
    dig = rng.integers(0, 1 << 62, (B, k, n)) % p
    if extremes:
        dig[0] = p[0] - 1
        dig[1, :, ::2] = 0
        dig[1, :, 1::2] = (p[0] - 1)[:, 0:1]
    adA = rng.integers(0, 1 << 62, (B, 2, k, n)) % p[:, None]
    adB = rng.integers(0, 1 << 62, (B + 3, 2, k, n)) % p[:, None]
    slot = rng.permutation(B + 3)[:B].astype(np.int32)
    d_dig = torch.from_numpy(dig.astype(np.int32)).cuda()
    d_adA = torch.from_numpy(adA.astype(np.int32)).cuda()
    d_adB = torch.from_numpy(adB.astype(np.int32)).cuda()
    d_slot = torch.from_numpy(slot).cuda()
    key = be.keys.galois[1]
    outs = []
    for aux in (False, True):
        out = torch.zeros((B + 3, 2, k, n), dtype=torch.int32, device="cuda")
        args = (d_dig.data_ptr(), stack, out[0, 0].data_ptr(), out[0, 1].data_ptr(), 2 * stack,
                d_slot.data_ptr(), d_adA[0, 0].data_ptr(), d_adA[0, 1].data_ptr(), 2 * stack,
                d_adB[0, 0].data_ptr(), d_adB[0, 1].data_ptr(), 2 * stack)
        if aux:
            per_ct = 9 * k * n
            cap = max(1, B // 3)  # force several chunks
            ws = torch.empty(cap * per_ct, dtype=torch.int32, device="cuda")
            ctx.call("hefv_keyswitch_aux", key.aux_dev.data_ptr(), args[0], args[1], None, 0,
                     *args[2:], ws.data_ptr(), cap, B, ctx.stream())
        else:
            ctx.call("hefv_keyswitch", key.body_dev.data_ptr(), key.mask_dev.data_ptr(), *args, B,
                     ctx.stream())
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    del galois_element
    return outs


@pytest.mark.parametrize("logn,k,B", [(14, 22, 9), (14, 24, 5), (13, 12, 7), (12, 17, 6), (11, 16, 5),
                                      (10, 9, 11)])
def test_aux_keyswitch_equals_per_prime(logn, k, B):
    direct, aux = _both(_params(logn, k), B, seed=logn * 100 + k, extremes=True)
    assert np.array_equal(direct, aux)


def test_aux_keyswitch_retina_profile_rotations_match_golden_path():
    """With the aux path on (default for retina), rotations equal the
    per-prime path bit for bit through the public API."""
    import os

    from oracle.fv_oracle import limb_digest
    from paper_1901_10074_b200.fv import FvBackend

    params = profile("retina")
    digs = []
    for flag in ("0", "1"):
        os.environ["HEFV_KS_AUX"] = flag
        try:
            be = FvBackend(params, rng=np.random.default_rng(5))
            assert be.ctx.ks_aux == (flag == "1")
            a = be.encrypt(np.arange(100))
            digs.append([limb_digest(be.rotate(a, r).parts) for r in (1, 3, 4095)]
                        + [limb_digest(be.mult(a, a).parts)])
        finally:
            os.environ.pop("HEFV_KS_AUX", None)
    assert digs[0] == digs[1]


@pytest.mark.parametrize("logn,k", [(14, 22), (12, 17)])
def test_aux_keyswitch_fused_automorphism_with_slot_map(logn, k):
    """Digits read through a slot map with the Galois automorphism applied in
    the load (hefv_keyswitch_aux dig_slot/galois) equal the per-prime kernel
    on materialised sigma_g(c1) rows (hefv_automorph)."""
    import torch

    from paper_1901_10074_b200.fv import FvBackend
    from paper_1901_10074_b200.ring import galois_element

    be = FvBackend(_params(logn, k), rng=np.random.default_rng(7))
    ctx = be.ctx
    n = ctx.n
    stack = k * n
    rng = np.random.default_rng(8)
    R, B = 9, 6
    p = np.array(ctx.q_primes, dtype=np.int64)[None, None, :, None]
    src = rng.integers(0, 1 << 62, (R, 2, k, n)) % p
    src[0, 1, :, ::3] = 0  # zero coefficients (sigma must keep them 0, not p)
    slot = rng.permutation(R)[:B].astype(np.int32)
    d_src = torch.from_numpy(src.astype(np.int32)).cuda()
    d_slot = torch.from_numpy(slot).cuda()
    off = 4 if logn == 14 else 2
    key = be.keys.galois[off]
    g = galois_element(off, n)
    outs = []
    for fused in (True, False):
        out = torch.zeros((R, 2, k, n), dtype=torch.int32, device="cuda")
        if fused:
            per_ct = 9 * stack
            ws = torch.empty(2 * per_ct, dtype=torch.int32, device="cuda")  # 2-ct chunks
            ctx.call("hefv_keyswitch_aux", key.aux_dev.data_ptr(), d_src[0, 1].data_ptr(),
                     2 * stack, d_slot.data_ptr(), g, out[0, 0].data_ptr(), out[0, 1].data_ptr(),
                     2 * stack, d_slot.data_ptr(), None, None, 0, None, None, 0, ws.data_ptr(),
                     2, B, ctx.stream())
        else:
            sig = torch.empty((B, 2, k, n), dtype=torch.int32, device="cuda")
            ctx.call("hefv_automorph", d_src.data_ptr(), 2 * stack, d_slot.data_ptr(),
                     sig.data_ptr(), 2, g, B, ctx.stream())
            ctx.call("hefv_keyswitch", key.body_dev.data_ptr(), key.mask_dev.data_ptr(),
                     sig[0, 1].data_ptr(), 2 * stack, out[0, 0].data_ptr(), out[0, 1].data_ptr(),
                     2 * stack, d_slot.data_ptr(), None, None, 0, None, None, 0, B, ctx.stream())
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
