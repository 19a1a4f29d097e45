"""One forward + one inverse batched NTT per bench configuration (the
ntt_microbench list of bench.py), for `ncu --set full -k regex:k_ntt`
digests of every size: python tools/ntt_profile_all.py"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch

from paper_1901_10074_b200 import _native as nat
from paper_1901_10074_b200.ring import find_ntt_primes, root_of_unity

lib = nat.load()
st = torch.cuda.current_stream().cuda_stream
for log_n, bits, L, batch in [(16, 60, 8, 64), (15, 55, 8, 128), (14, 60, 8, 256),
                              (13, 60, 8, 256), (12, 50, 8, 1024), (14, 30, 22, 256),
                              (12, 30, 8, 1024)]:
    n = 1 << log_n
    primes = find_ntt_primes(L, bits, 2 * n)
    psis = [root_of_unity(p, n) for p in primes]
    h = C.c_void_p()
    if bits > 30:
        nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 0, None, None, L,
                                      (C.c_uint64 * L)(*primes), (C.c_uint64 * L)(*psis)))
        x = torch.randint(0, 1 << 40, (batch, L, n), dtype=torch.int64, device="cuda")
        f, g = lib.hefv_ntt_fwd64, lib.hefv_ntt_inv64
    else:
        nat.check(lib.hefv_ctx_create(C.byref(h), log_n, L, (C.c_uint32 * L)(*primes),
                                      (C.c_uint32 * L)(*psis), 0, None, None))
        x = torch.randint(0, 1 << 29, (batch, L, n), dtype=torch.int32, device="cuda")
        f, g = lib.hefv_ntt_fwd32, lib.hefv_ntt_inv32
    y = torch.empty_like(x)
    nat.check(f(h, x.data_ptr(), y.data_ptr(), batch, L, 0, 0, st))
    nat.check(g(h, y.data_ptr(), x.data_ptr(), batch, L, 0, 0, st))
    torch.cuda.synchronize()
    print(f"N=2^{log_n} {bits}-bit L={L} batch={batch}: fwd+inv done", flush=True)
    lib.hefv_ctx_destroy(h)
