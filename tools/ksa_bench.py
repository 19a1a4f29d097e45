"""Aux-basis key switch (the config-2 hot path) microbenchmark and ncu target:
B ciphertexts rotated by one hop (fused Galois automorphism) through
planner.rotation_keyswitch, timed with CUDA events.

python tools/ksa_bench.py [profile] [B] [iters]
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import planner
from paper_1901_10074_b200.fv import FvBackend
from paper_1901_10074_b200.params import profile
from paper_1901_10074_b200.ring import galois_element

name = sys.argv[1] if len(sys.argv) > 1 else "retina"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if name.startswith("config"):
    from paper_1901_10074_b200.configs import config_params

    p = config_params(int(name[6:]))
else:
    p = profile(name)
be = FvBackend(p, rng=np.random.default_rng(1))
ctx = be.ctx
assert ctx.ks_aux, "profile does not use the aux-basis key switch"
k, n = ctx.k, ctx.n
stack = k * n
gen = torch.Generator(device="cuda").manual_seed(1)
pr = torch.tensor(ctx.q_primes, dtype=torch.int64, device="cuda").view(1, 1, k, 1)
src = (torch.randint(0, 1 << 31, (B, 2, k, n), dtype=torch.int64, device="cuda", generator=gen)
       % pr).to(torch.int32)
out = torch.empty_like(src)
scr = torch.empty(B * stack, dtype=torch.int32, device="cuda")
key = be.keys.galois[1]
g = galois_element(1, n)


def hop():
    planner.rotation_keyswitch(ctx, key, src.data_ptr(), 2 * stack, None, g, B, out.data_ptr(),
                               out.data_ptr() + stack * 4, 2 * stack, None, None, None, 0,
                               scr.data_ptr())


hop()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    hop()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
print(f"rotation hop (automorph + aux key switch), B={B}: {ms:.3f} ms per launch, "
      f"{1000 * ms / B:.2f} us per ciphertext", flush=True)
