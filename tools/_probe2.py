import sys
sys.path.insert(0, ".")
from tools.probe_int import measure
for k in (0, 10, 11, 12):
    print(k, round(measure(k) / 1e12, 3), "T/s", flush=True)
