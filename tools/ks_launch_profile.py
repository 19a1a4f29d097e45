"""Per-launch key-switch batch sizes and times for one config-2 inference
(CUDA events around every keyswitch_call): where small batches cost.

python tools/ks_launch_profile.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200 import planner
from paper_1901_10074_b200.configs import KEY_SEED, config_network, config_params
from paper_1901_10074_b200.fv import FvBackend

params = config_params(2)
img, net = config_network(2)
be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
pv = I.pack_image(be, img)
I.infer(be, net, pv)
torch.cuda.synchronize()
planner.KS_EVENTS = []
I.infer(be, net, pv)
torch.cuda.synchronize()
ev = [(a.elapsed_time(b), n) for a, b, n in planner.KS_EVENTS]
planner.KS_EVENTS = None
tot = sum(t for t, _ in ev)
buckets = {}
for t, n in ev:
    key = 1 << max(0, (n - 1).bit_length() - 1)
    b = buckets.setdefault(key, [0, 0, 0.0])
    b[0] += 1
    b[1] += n
    b[2] += t
print(f"{len(ev)} launches, {sum(n for _, n in ev)} cts, {tot:.1f} ms")
for key in sorted(buckets):
    c, n, t = buckets[key]
    print(f"B in [{key},{2 * key}): {c:4d} launches {n:7d} cts {t:9.1f} ms  {1000 * t / n:7.2f} us/ct")
