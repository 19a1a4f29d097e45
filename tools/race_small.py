"""Small workload for compute-sanitizer racecheck / memcheck: every CTA-resident
transform kernel (30-bit batched, 64-bit one-kernel and split forms) and the
aux-basis key switch at a small and at the retina ring dimension.

compute-sanitizer --tool racecheck python tools/race_small.py [quick]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import _native as nat
from paper_1901_10074_b200.fv import FvBackend
from paper_1901_10074_b200.params import BackendParams, profile
from paper_1901_10074_b200.ring import find_ntt_primes, root_of_unity

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
lib = nat.load()
st = torch.cuda.current_stream().cuda_stream
# standalone transforms: round trips must reproduce the input
for log_n, bits in ((12, 30), (14, 30), (12, 50), (13, 60), (14, 60), (15, 55), (16, 60)):
    if quick and log_n > 14:
        continue
    n, L = 1 << log_n, 2
    primes = find_ntt_primes(L, bits, 2 * n)
    psis = [root_of_unity(p, n) for p in primes]
    h = C.c_void_p()
    if bits <= 30:
        nat.check(lib.hefv_ctx_create(C.byref(h), log_n, L, (C.c_uint32 * L)(*primes),
                                      (C.c_uint32 * L)(*psis), 0, None, None))
        x = torch.randint(0, min(primes), (3, L, n), dtype=torch.int32, device="cuda")
        y, z = torch.empty_like(x), torch.empty_like(x)
        nat.check(lib.hefv_ntt_fwd32(h, x.data_ptr(), y.data_ptr(), 3, L, 0, 0, st))
        nat.check(lib.hefv_ntt_inv32(h, y.data_ptr(), z.data_ptr(), 3, L, 0, 0, st))
    else:
        nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 0, None, None, L,
                                      (C.c_uint64 * L)(*primes), (C.c_uint64 * L)(*psis)))
        x = torch.randint(0, min(primes), (3, L, n), dtype=torch.int64, device="cuda")
        y, z = torch.empty_like(x), torch.empty_like(x)
        nat.check(lib.hefv_ntt_fwd64(h, x.data_ptr(), y.data_ptr(), 3, L, 0, 0, st))
        nat.check(lib.hefv_ntt_inv64(h, y.data_ptr(), z.data_ptr(), 3, L, 0, 0, st))
    torch.cuda.synchronize()
    print(f"ntt 2^{log_n} {bits}-bit round trip", bool(torch.equal(x, z)), flush=True)
    lib.hefv_ctx_destroy(h)
profiles = [BackendParams(ring_dimension=1024, coeff_modulus_bits=300, plain_modulus=12289,
                          slot_count=512, depth_budget=4)]
if not quick:
    profiles.append(profile("retina"))
for p in profiles:
    be = FvBackend(p, rng=np.random.default_rng(1))
    v = np.arange(p.slot_count) % 7
    a = be.encrypt(v)
    b = be.rotate(a, 3)
    c = be.cmult(a, v)
    d = be.mult(a, a)
    print(p.ring_dimension, np.array_equal(be.decrypt(b), np.roll(v, -3)), flush=True)
