"""The tcgen05 int8 plumbing of csrc/umma.cuh (descriptors, MMA, TMEM) that
the tensor-core contraction experiment used (tools/experiments/): C = A B^T
for u8 operands in the interleaved and the 128-byte-swizzled K-major
layouts, equal to numpy's exact int64 product."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ks,swizzle,m64", [(1, 0, False), (3, 0, False), (3, 1, False),
                                            (2, 1, False), (3, 0, True)])
def test_umma_u8_exact(ks, swizzle, m64):
    import torch

    from paper_1901_10074_b200 import _native as nat

    lib = nat.load()
    rng = np.random.default_rng(ks * 10 + swizzle)
    K = 32 * ks
    A = rng.integers(0, 256, (128, K), dtype=np.uint8)
    if m64:
        A[64:] = 0
    B = rng.integers(0, 256, (256, K), dtype=np.uint8)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.full((128, 256), -1, dtype=torch.int32, device="cuda")
    code = (ks + 8 * swizzle) * (-1 if m64 else 1)
    nat.check(lib.hefv_probe_umma(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), code,
                                  torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = dC.cpu().numpy().astype(np.int64)
    want = A.astype(np.int64) @ B.astype(np.int64).T
    if m64:  # M = 64 places row r in TMEM lane (r % 16) + 32 (r / 16)
        lanes = [(r % 16) + 32 * (r // 16) for r in range(64)]
        assert np.array_equal(got[lanes], want[:64])
    else:
        assert np.array_equal(got, want)


def test_tmem_load_shapes_and_mma_timing_probes():
    """The measurement probes behind DESIGN.md's tensor-core numbers run:
    32x32b stores read back through the 16x64b / 16x256b shapes with the
    lane / column placement the epilogue design relied on, and the MMA
    timing probe returns a positive cycle count."""
    import torch

    from paper_1901_10074_b200 import _native as nat

    lib = nat.load()
    st = torch.cuda.current_stream().cuda_stream
    d = torch.zeros(128, dtype=torch.int32, device="cuda")
    nat.check(lib.hefv_probe_tmem_shape(d.data_ptr(), 2, st))  # 16x256b.x1
    torch.cuda.synchronize()
    v = d.cpu().numpy().reshape(32, 4)
    for t in range(32):  # thread t: lanes t/4 and t/4 + 8, columns 2 (t%4), +1
        r, c = t // 4, 2 * (t % 4)
        assert list(v[t]) == [1000 * r + c, 1000 * r + c + 1, 1000 * (r + 8) + c,
                              1000 * (r + 8) + c + 1]
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    nat.check(lib.hefv_probe_umma_lat(cyc.data_ptr(), 16, 3, -1, st))
    torch.cuda.synchronize()
    assert cyc.item() > 0


def test_integer_pipe_probes_run():
    import torch

    from paper_1901_10074_b200 import _native as nat

    lib = nat.load()
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    for kind in range(10):
        nat.check(lib.hefv_probe_int(kind, 148, 2, out.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
