"""Per-layer device time of one encrypted inference, split into key-switch
time (library-side CUDA events around every key-switch call) and the rest.

python tools/layer_times.py [config]      (default 3)
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200 import planner
from paper_1901_10074_b200.configs import KEY_SEED, config_network, config_params
from paper_1901_10074_b200.fv import FvBackend

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
params = config_params(cfg)
img, net = config_network(cfg)
be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
pv = I.pack_image(be, img)
torch.cuda.synchronize()
rows = []
for layer in net.layers:
    planner.ks_reset(be.ctx, timing=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if isinstance(layer, I.SquareSpec):
        nxt = I.square_activation(be, pv)
    else:
        nxt = I.layer_eval(be, I._compiled_rows(layer, pv.slots_used), pv,
                           scale_factor=1 << layer.scale_bits)
    e1.record()
    torch.cuda.synchronize()
    ks = planner.ks_stats(be.ctx)
    ms = e0.elapsed_time(e1)
    rows.append({"layer": type(layer).__name__, "in_cts": len(pv.cts), "out_cts": len(nxt.cts),
                 "ms": round(ms, 1), "ks_ms": round(ks["ks_ms"], 1),
                 "other_ms": round(ms - ks["ks_ms"], 1), "ks_calls": ks["ks_launches"],
                 "ks_cts": ks["ks_cts"],
                 "us_per_ks": round(1000 * ks["ks_ms"] / max(1, ks["ks_cts"]), 2)})
    pv = nxt
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"total_ms": round(sum(r["ms"] for r in rows), 1),
                  "ks_ms": round(sum(r["ks_ms"] for r in rows), 1)}))
