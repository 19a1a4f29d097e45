"""Quick timing of one encrypted inference (development tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import config_network, config_params
from paper_1901_10074_b200.fv import FvBackend

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t0 = time.time()
img, net = config_network(cfg)
be = FvBackend(config_params(cfg), rng=np.random.default_rng(1234))
torch.cuda.synchronize(); t1 = time.time()
print(f"keygen {t1-t0:.2f}s", flush=True)
for it in range(2):
    torch.cuda.synchronize(); a = time.time()
    pv = I.pack_image(be, img)
    torch.cuda.synchronize(); b = time.time()
    cur = pv
    for li, layer in enumerate(net.layers):
        torch.cuda.synchronize(); l0 = time.time()
        if isinstance(layer, I.SquareSpec):
            cur = I.square_activation(be, cur)
        else:
            rows = I.compile_conv(layer, cur.slots_used) if isinstance(layer, I.ConvSpec) else I.compile_fc(layer, cur.slots_used)
            l1 = time.time()
            cur = I.layer_eval(be, rows, cur)
        torch.cuda.synchronize(); print(f"  layer {li} {type(layer).__name__} {time.time()-l0:.3f}s", flush=True)
    logits = I.decrypt_logits(be, cur)
    c = time.time()
    print(f"iter {it}: encrypt {b-a:.3f}s total {c-a:.3f}s logits {logits}", flush=True)
print(be.cost_report())
