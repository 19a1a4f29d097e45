"""tcgen05 int8 tensor-core checks (development aid): C = A x B^T for random
u8 operands vs numpy (interleaved and 128-byte-swizzled operand layouts,
M = 128 and 64), the TMEM lane placement of M = 64, TMEM load shapes, and
MMA latency / throughput (python tools/umma_check.py)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import _native as nat

lib = nat.load()
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
rng = np.random.default_rng(1)
for ks, sw in ((1, 0), (3, 0), (3, 1), (2, 1)):
    K = 32 * ks
    A = rng.integers(0, 256, (128, K), dtype=np.uint8)
    B = rng.integers(0, 256, (256, K), dtype=np.uint8)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros((128, 256), dtype=torch.int32, device="cuda")
    nat.check(lib.hefv_probe_umma(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), ks + 8 * sw, st()))
    torch.cuda.synchronize()
    want = A.astype(np.int64) @ B.astype(np.int64).T
    got = dC.cpu().numpy().astype(np.int64)
    bad = np.argwhere(got != want)
    print(f"ks={ks} swizzle={sw}: {'OK' if len(bad) == 0 else f'{len(bad)} mismatches'}")
for shape, name in ((0, "M64 N128"), (1, "M128 N128"), (2, "M128 N256"), (3, "M64 N256")):
    for chain, depth in ((3, 1), (3, 4), (12, 2)):
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        reps = 200
        code = depth + 4 * shape
        nat.check(lib.hefv_probe_umma_lat(d.data_ptr(), reps, chain, -code, st()))
        torch.cuda.synchronize()
        M, N = (64 if shape in (0, 3) else 128), (128 if shape < 2 else 256)
        cyc = d.item() / reps / chain
        print(f"{name} chain {chain} depth {depth}: {cyc:.0f} cycles per MMA, "
              f"{M * N * 32 / cyc:.0f} MACs/clk")
