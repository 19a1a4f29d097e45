"""Whole-network limb parity of the batched planner against the per-op GPU
path, at a config's real size (development / evidence run; the test suite
covers config 2 in full and config 3 by a conv1 tile + the conv2/square/FC
tail, tests/test_gpu_network.py -- this runs EVERY row of EVERY layer):

python tools/network_parity.py [config] [images] > gpurun_out/network_parity_cN.json

(config 5: the first ``images`` images of the 256-image stream, default 4, one
backend and one Generator across the stream as in the reference's batch run.)

The network runs twice from the same seed: through ``layer_eval`` /
``square_activation`` (the planner: whole layers as batched launches) and
through the reference's per-row loop replayed op by op (``_serial_layer_eval``
+ ``mult``; inference.py:277-349 of the reference), whose primitives are each
pinned to reference digests (tests/test_gpu_ops.py).  Compared: the sha256 of
every output ciphertext's int64 limbs after each layer, the levels, the
CostReport and the decrypted logits (also against the exact plaintext forward
pass).  Config 3: 142,386 rows, 2,780,236 key-switch hops per run.
"""
import gc
import hashlib
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import (batch_images, centred_mod, config_network,
                                           config_params, plaintext_forward)
from paper_1901_10074_b200.fv import FvBackend


def digest(parts) -> str:
    h = hashlib.sha256()
    for p in parts:
        h.update(np.ascontiguousarray(np.asarray(p, dtype=np.int64)).astype("<i8").tobytes())
    return h.hexdigest()


def run_image(be, net, img, planned: bool, tag: str):
    """One image through every layer; (per-layer trace, logits, seconds)."""
    pv = I.pack_image(be, img)
    trace, times = [], []
    cur = pv
    for layer in net.layers:
        t0 = time.perf_counter()
        if isinstance(layer, I.SquareSpec):
            if planned:
                nxt = I.square_activation(be, cur)
            else:
                nxt = I.PackedVector(cur.logical_length, cur.slots_used,
                                     [be.mult(ct, ct) for ct in cur.cts],
                                     scale=cur.scale * cur.scale, shape=cur.shape)
        else:
            rows = (I.compile_conv(layer, cur.slots_used) if isinstance(layer, I.ConvSpec)
                    else I.compile_fc(layer, cur.slots_used))
            nxt = (I.layer_eval(be, rows, cur) if planned
                   else I._serial_layer_eval(be, rows, cur, True, 1))
        torch.cuda.synchronize()
        times.append(round(time.perf_counter() - t0, 2))
        if cur is not pv:
            be.release(*cur.cts)
        cur = nxt
        trace.append({"layer": tag + type(layer).__name__, "cts": len(cur.cts),
                      "levels": [ct.level_used for ct in cur.cts],
                      "digests": [digest(ct.parts) for ct in cur.cts]})
        print(f"  {'planner' if planned else 'per-op'} {tag}{type(layer).__name__}: {times[-1]} s",
              file=sys.stderr, flush=True)
    logits = [int(v) for v in I.decrypt_logits(be, cur)]
    be.release(*pv.cts, *cur.cts)
    return trace, logits, times


def run(cfg: int, planned: bool, images: int):
    img, net = config_network(2 if cfg == 5 else cfg)
    params = config_params(cfg)
    stream = batch_images(images) if cfg == 5 else [img]
    be = FvBackend(params, rng=np.random.default_rng(1234))
    trace, logits, want, times = [], [], [], []
    for n, im in enumerate(stream):
        tr, lg, tm = run_image(be, net, im, planned, f"image{n}." if cfg == 5 else "")
        trace += tr
        logits += lg
        times += tm
        want += [int(v) for v in centred_mod(plaintext_forward(net, im), params.plain_modulus)]
    cost = be.cost_report().as_dict()
    del be
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return trace, cost, logits, want, times


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    images = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    tp, cp, lp, want, timep = run(cfg, True, images)
    ts, cs, ls, _, times = run(cfg, False, images)
    layers = []
    for a, b in zip(tp, ts):
        layers.append({"layer": a["layer"], "cts": a["cts"], "levels": a["levels"],
                       "limbs_equal": a["digests"] == b["digests"],
                       "levels_equal": a["levels"] == b["levels"],
                       "digest_of_digests": hashlib.sha256("".join(a["digests"]).encode()).hexdigest()})
    ok = (all(x["limbs_equal"] and x["levels_equal"] for x in layers) and cp == cs and lp == ls
          and lp == want and len(tp) == len(ts))
    print(json.dumps({
        "config": cfg, "images": images if cfg == 5 else 1, "all_equal": ok, "layers": layers,
        "cost_report_equal": cp == cs, "cost_report": cp,
        "logits_planner": lp, "logits_per_op": ls, "logits_plaintext_forward": want,
        "layer_seconds": {"planner": timep, "per_op": times},
        "gpu": torch.cuda.get_device_name(0),
    }))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
