"""cProfile of one config-2 encrypted inference on the GPU (host-side view:
how much of the step the host spends outside the blocking launches).

python tools/prof_infer.py
"""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import KEY_SEED, config_network, config_params
from paper_1901_10074_b200.fv import FvBackend
params = config_params(2); img, net = config_network(2)
be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
pv = I.pack_image(be, img); torch.cuda.synchronize()
I.infer(be, net, pv); torch.cuda.synchronize()
pr = cProfile.Profile(); t0 = time.perf_counter(); pr.enable()
out = I.infer(be, net, pv); torch.cuda.synchronize()
pr.disable(); print("wall", time.perf_counter() - t0)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
