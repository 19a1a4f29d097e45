"""64-bit key switch (config 4) microbenchmark / ncu target.
python tools/ks64_bench.py LOGN L bits B [path] [iters]"""
import sys

sys.path.insert(0, ".")
import torch

from paper_1901_10074_b200.ring import find_ntt_primes
from paper_1901_10074_b200.rns import RnsKeySwitch64

log_n, L, bits, B = (int(v) for v in sys.argv[1:5])
path = sys.argv[5] if len(sys.argv) > 5 else "aux"
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
n = 1 << log_n
primes = find_ntt_primes(L, bits, 2 * n)
ks = RnsKeySwitch64(primes, n, aux=(path == "aux"))
key = ks.random_key(1)
p = torch.tensor(primes, dtype=torch.int64, device="cuda").view(1, L, 1)
dig = torch.randint(0, 1 << 62, (B, L, n), dtype=torch.int64, device="cuda") % p
ks.switch(key, dig, path)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(iters):
    ks.switch(key, dig, path)
b.record()
torch.cuda.synchronize()
t = a.elapsed_time(b) / iters / 1e3
mm = (L * L + 2 * L) * ((n // 2) * log_n + n) + 2 * L * L * n
print(f"N=2^{log_n} L={L} {bits}-bit B={B} {path}: {t / B * 1e6:.2f} us/ct, "
      f"{mm * B / t / 1e12:.3f} T ref-modmul/s", flush=True)
