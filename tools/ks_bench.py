"""Key-switch / NTT kernel microbenchmark (development + ncu target).

python tools/ks_bench.py [profile] [B] [iters]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200.fv import FvBackend
from paper_1901_10074_b200.params import profile
from paper_1901_10074_b200.ring import galois_element

name = sys.argv[1] if len(sys.argv) > 1 else "retina"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
p = profile(name)
be = FvBackend(p, rng=np.random.default_rng(1))
ctx = be.ctx
k, n = ctx.k, ctx.n
stack = k * n
acc = torch.randint(0, 1 << 29, (B, 2, k, n), dtype=torch.int32, device="cuda")
scr = torch.empty_like(acc)
key = be.keys.galois[1]
st = ctx.stream()
g = galois_element(1, n)
a0 = acc.data_ptr(); a1 = a0 + stack * 4; s0 = scr.data_ptr(); s1 = s0 + stack * 4


def ks():
    ctx.call("hefv_keyswitch", key.body_dev.data_ptr(), key.mask_dev.data_ptr(), s1, 2 * stack,
             a0, a1, 2 * stack, None, s0, None, 2 * stack, a0, a1, 2 * stack, B, st)


def aut():
    ctx.call("hefv_automorph", a0, 2 * stack, None, s0, 2, g, B, st)


def ntt():
    ctx.call("hefv_ntt_fwd32", s0, a0, B * 2, k, 0, 0, st)


for name_, fn in (("automorph", aut), ("keyswitch", ks), ("ntt_fwd32 (2k polys per ct)", ntt)):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"{name_}: {ms:.3f} ms per launch, {1000 * ms / B:.2f} us per ciphertext", flush=True)
