"""Top SASS instructions of one kernel in an ncu report by a chosen column
(development aid): python tools/ncu_sass_hot.py REPORT KERNEL_REGEX [COLUMN] [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
ci = h.index(col)
def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


data = [r for r in rows[2:] if len(r) == len(h) and num(r[ci] or "0") is not None]
tot = sum(num(r[ci] or '0') for r in data)
print(f"{col}: total {tot:.0f}")
for r in sorted(data, key=lambda r: -num(r[ci] or '0'))[:top]:
    print(f"{num(r[ci] or '0'):10.0f} {r[0]} {r[1][:70]}")
