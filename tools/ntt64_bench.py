"""Batched 64-bit-prime NTT throughput (device order), limb-polys/s and the
roofline fraction against the measured 64-bit lazy-butterfly rate.

python tools/ntt64_bench.py [LOGN] [bits] [L] [batch] [iters]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch

from paper_1901_10074_b200 import _native as nat
from paper_1901_10074_b200.ring import find_ntt_primes, root_of_unity

log_n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 60
L = int(sys.argv[3]) if len(sys.argv) > 3 else 8
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 256
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 10
PEAK64 = 0.845  # measured lazy 64-bit Shoup butterflies/s (T), tools/probe_int.py
lib = nat.load()
n = 1 << log_n
primes = find_ntt_primes(L, bits, 2 * n)
psis = [root_of_unity(p, n) for p in primes]
h = C.c_void_p()
nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 0, None, None, L, (C.c_uint64 * L)(*primes),
                              (C.c_uint64 * L)(*psis)))
x = torch.randint(0, 1 << 40, (batch, L, n), dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
work = (n // 2) * log_n + n
for fn, name in ((lib.hefv_ntt_fwd64, "fwd"), (lib.hefv_ntt_inv64, "inv")):
    src, dst = (x, y) if name == "fwd" else (y, x)
    nat.check(fn(h, src.data_ptr(), dst.data_ptr(), batch, L, 0, 0, st))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        nat.check(fn(h, src.data_ptr(), dst.data_ptr(), batch, L, 0, 0, st))
    b.record()
    torch.cuda.synchronize()
    ps = batch * L / (a.elapsed_time(b) / iters * 1e-3)
    print(f"N=2^{log_n} {bits}-bit L={L} batch={batch} {name}: {ps / 1e6:.3f} M polys/s, "
          f"{ps * work / 1e12:.3f} Tbfly/s, frac {ps * work / 1e12 / PEAK64:.3f}", flush=True)
lib.hefv_ctx_destroy(h)
