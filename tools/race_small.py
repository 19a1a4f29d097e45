"""Small workload for compute-sanitizer racecheck: every CTA-resident transform kernel."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1901_10074_b200.fv import FvBackend
from paper_1901_10074_b200.params import BackendParams, profile
for p in (BackendParams(ring_dimension=1024, coeff_modulus_bits=90, plain_modulus=12289,
                        slot_count=512, depth_budget=4), profile("retina")):
    be = FvBackend(p, rng=np.random.default_rng(1))
    v = np.arange(p.slot_count) % 7
    a = be.encrypt(v)
    b = be.rotate(a, 3)
    c = be.cmult(a, v)
    d = be.mult(a, a)
    print(p.ring_dimension, np.array_equal(be.decrypt(b), np.roll(v, -3)), flush=True)
