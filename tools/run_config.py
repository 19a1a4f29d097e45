"""Time whole encrypted inferences of a config on the GPU and check the
decrypted logits against the exact plaintext forward pass (mod t).

  python tools/run_config.py 3            # DR-shaped 256x256x3 net, once
  python tools/run_config.py 5 --images 4 # config 5 sample: images/s
Prints one JSON line.
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200 import planner
from paper_1901_10074_b200.configs import (KEY_SEED, batch_images, centred_mod, config_network,
                                           config_params, plaintext_forward, workload_op_counts)
from paper_1901_10074_b200.fv import FvBackend

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--images", type=int, default=1)
args = ap.parse_args()
cfg = args.config
params = config_params(cfg)
img0, net = config_network(cfg)
t0 = time.perf_counter()
be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
torch.cuda.synchronize()
keygen = time.perf_counter() - t0
images = [img0] if cfg != 5 else batch_images(args.images)
res = {"config": cfg, "profile": params.name, "q_primes": be.ctx.k, "aux_primes": be.ctx.a,
       "keygen_s": round(keygen, 2), "images": len(images)}
lat = []
ok = True
for img in images:
    torch.cuda.synchronize()
    planner.ks_reset(be.ctx)
    a = time.perf_counter()
    out = I.infer(be, net, I.pack_image(be, img))
    logits = I.decrypt_logits(be, out)
    torch.cuda.synchronize()
    lat.append(time.perf_counter() - a)
    want = centred_mod(plaintext_forward(net, img), params.plain_modulus)
    ok = ok and [int(v) for v in logits] == want
    ks = planner.ks_stats(be.ctx)
res.update({"latency_s": [round(x, 3) for x in lat], "images_per_s": round(len(lat) / sum(lat), 5),
            "logits_equal_exact_plaintext_mod_t": ok, "ks_launches_per_image": ks["ks_launches"],
            "ks_cts_per_image": ks["ks_cts"],
            "cost_report": be.cost_report().as_dict(),
            "serial_op_counts": workload_op_counts(cfg if cfg != 5 else 2)})
print(json.dumps(res), flush=True)
