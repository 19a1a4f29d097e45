"""Key-switch throughput at arbitrary (N, k): us per ciphertext and the
algorithmic modmul rate M / t, M = (k^2 + 2k)((N/2) log2 N + N) + 2 k^2 N.

python tools/ks_shape_probe.py LOGN K [B] [iters]
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200.fv import FvBackend
from paper_1901_10074_b200.params import BackendParams
from paper_1901_10074_b200.ring import find_ntt_primes

logn, k = int(sys.argv[1]), int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 5
n = 1 << logn
t = find_ntt_primes(1, 40, 2 * n)[0]
p = BackendParams(ring_dimension=n, coeff_modulus_bits=30 * k, plain_modulus=t, slot_count=n // 2,
                  depth_budget=4)
be = FvBackend(p, rng=np.random.default_rng(1))
ctx = be.ctx
stack = k * n
acc = torch.randint(0, 1 << 29, (B, 2, k, n), dtype=torch.int32, device="cuda")
scr = torch.empty_like(acc)
key = be.keys.galois[1]
st = ctx.stream()
a0 = acc.data_ptr()
a1 = a0 + stack * 4
s0 = scr.data_ptr()
s1 = s0 + stack * 4


ws = None
if key.aux_dev is not None:
    per_ct = 9 * k * n
    import os

    cap = max(1, min(B, int(float(os.environ.get("KS_WS_GB", "6")) * (1 << 30)) // (4 * per_ct)))
    ws = torch.empty(cap * per_ct, dtype=torch.int32, device="cuda")


def ks():
    args = (s1, 2 * stack, a0, a1, 2 * stack, None, s0, None, 2 * stack, a0, a1, 2 * stack)
    if ws is not None:
        ctx.call("hefv_keyswitch_aux", key.aux_dev.data_ptr(), args[0], args[1], None, 0,
                 *args[2:], ws.data_ptr(), cap, B, st)
    else:
        ctx.call("hefv_keyswitch", key.body_dev.data_ptr(), key.mask_dev.data_ptr(), *args, B, st)


ks()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ks()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / iters * 1000 / B
M = (k * k + 2 * k) * ((n // 2) * logn + n) + 2 * k * k * n
mode = "aux" if ws is not None else "per-prime"
print(f"N=2^{logn} k={k} B={B} [{mode}]: {us:.2f} us/ct, {M / us / 1e6:.3f} Tmodmul/s-equivalent",
      flush=True)
