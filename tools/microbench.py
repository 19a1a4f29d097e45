"""Config 4 microbench: batched forward/inverse negacyclic RNS-NTT and a full
key switch over L NTT-friendly primes of 50-60 bits, N = 2^12..2^16.

  python tools/microbench.py [--quick]   -> one JSON object on stdout

Throughput is limb-polys/s (one polynomial under one prime) for the NTTs and
ciphertexts/s for the key switch (B ciphertexts of L limbs switched under one
key).  Roofline: a transform of N points is (N/2) log2 N butterflies + N
merged twist products; the peak is the measured lazy-Shoup butterfly rate of
tools/probe_int.py (64-bit butterflies cost ~3x the 32-bit one: reported as
a fraction of the 32-bit rate / 3 as well), and the HBM bound is 2 N w bytes
per transform (in + out).
"""

import argparse
import ctypes as C
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1901_10074_b200 import _native as nat
from paper_1901_10074_b200.ring import find_ntt_primes, root_of_unity
from paper_1901_10074_b200.rns import RnsKeySwitch64


def timeit(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters / 1e3  # seconds


def ntt_case(log_n, bits, L, batch):
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
    tf = timeit(lambda: nat.check(lib.hefv_ntt_fwd64(h, x.data_ptr(), y.data_ptr(), batch, L, 0, 0, st)))
    ti = timeit(lambda: nat.check(lib.hefv_ntt_inv64(h, y.data_ptr(), x.data_ptr(), batch, L, 0, 0, st)))
    lib.hefv_ctx_destroy(h)
    polys = batch * L
    bfly = (n // 2) * log_n + n
    return {"fwd_polys_s": round(polys / tf, 1), "inv_polys_s": round(polys / ti, 1),
            "fwd_Tbfly_s": round(polys * bfly / tf / 1e12, 4),
            "fwd_hbm_GBs": round(polys * 2 * n * 8 / tf / 1e9, 1)}


def ks_case(log_n, bits, L, B):
    n = 1 << log_n
    primes = find_ntt_primes(L, bits, 2 * n)
    ks = RnsKeySwitch64(primes, n)
    key = ks.random_key(1)
    p = torch.tensor(primes, dtype=torch.int64, device="cuda").view(1, L, 1)
    dig = torch.randint(0, 1 << 62, (B, L, n), dtype=torch.int64, device="cuda") % p
    t = timeit(lambda: ks.switch(key, dig), iters=3)
    modmuls = (L * L + 2 * L) * ((n // 2) * log_n + n) + 2 * L * L * n
    return {"cts_s": round(B / t, 1), "us_per_ct": round(t / B * 1e6, 2),
            "Tmodmul_s": round(modmuls * B / t / 1e12, 4),
            "path": "aux" if ks.aux else "direct"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, "tools")
    from probe_int import measure

    peak = measure(4) / 1e12
    out = {"peak_shoup32_Tbfly_s": round(peak, 3), "ntt": {}, "keyswitch": {}}
    logns = [12, 14, 16] if args.quick else [12, 13, 14, 15, 16]
    for log_n in logns:
        for L in ([1, 8] if args.quick else [1, 2, 4, 8]):
            for bits in (50, 60):
                for batch in ([64] if args.quick else [1, 8, 64, 256]):
                    if batch * L * (1 << log_n) * 8 > (2 << 30):
                        continue
                    key = f"N=2^{log_n},L={L},{bits}bit,batch={batch}"
                    out["ntt"][key] = ntt_case(log_n, bits, L, batch)
            for bits in (50, 60):
                # batch: as many ciphertexts as a 256 MB scratch holds, up to 1024
                # (small L needs large batches to fill the GPU)
                B = max(1, min(1024, (1 << 28) // (L * L * (1 << log_n) * 8)))
                out["keyswitch"][f"N=2^{log_n},L={L},{bits}bit,B={B}"] = ks_case(log_n, bits, L, B)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
