"""Time the paper's interleaved (per-pixel broadcast) baseline on the GPU
backend for a config's network and check the logits against the exact
plaintext forward pass (mod t).  The paper's comparison: compact packing
(bench.py / tools/run_config.py) vs this.

  python tools/run_interleaved.py 2      # ROP: 9,216 pixel ciphertexts
Prints one JSON line with per-stage seconds.
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import (KEY_SEED, centred_mod, config_network, config_params,
                                           plaintext_forward)
from paper_1901_10074_b200.fv import FvBackend

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
args = ap.parse_args()
params = config_params(args.config)
img, net = config_network(args.config)
be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
torch.cuda.synchronize()
stages = {}
a = time.perf_counter()
px = I.pack_image_interleaved(be, img)
torch.cuda.synchronize()
stages["encrypt_pixels_s"] = time.perf_counter() - a
vals = px
for li, layer in enumerate(net.layers):
    b = time.perf_counter()
    if isinstance(layer, I.SquareSpec):
        from paper_1901_10074_b200.broadcast import square_layer

        out = square_layer(be, vals)
    else:
        rows = (I.compile_conv(layer, slots_used=layer.in_len) if isinstance(layer, I.ConvSpec)
                else I.compile_fc(layer, slots_used=layer.in_len))
        from paper_1901_10074_b200.broadcast import broadcast_layer_eval

        out = broadcast_layer_eval(be, rows, vals)
        be.release(*vals)
    vals = out
    torch.cuda.synchronize()
    stages[f"layer{li}_{type(layer).__name__}_s"] = time.perf_counter() - b
c = time.perf_counter()
logits = I.decrypt_logits(be, vals)
stages["decrypt_s"] = time.perf_counter() - c
total = time.perf_counter() - a
want = centred_mod(plaintext_forward(net, img), params.plain_modulus)
res = {"config": args.config, "packing": "interleaved", "pixels": len(px),
       "stages": {k: round(v, 3) for k, v in stages.items()}, "latency_s": round(total, 3),
       "latency_excl_pixel_encryption_s": round(total - stages["encrypt_pixels_s"], 3),
       "logits_equal_exact_plaintext_mod_t": [int(v) for v in logits] == want,
       "cost_report": be.cost_report().as_dict(),
       "peak_hbm_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)}
print(json.dumps(res), flush=True)
