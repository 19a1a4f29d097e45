"""Warp-stall samples of one kernel in an ncu --set full --import-source on report,
aggregated by SASS opcode and stall reason (development aid):
python tools/ncu_stalls_by_opcode.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
seen, uniq = set(), []
for r in data:  # a report with several launches of the kernel repeats every address
    if r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)


def f(r, c):
    try:
        return float(r[h.index(c)].replace(",", ""))
    except ValueError:
        return 0.0


st = ["stall_not_selected", "stall_math", "stall_wait", "stall_dispatch", "stall_long_sb",
      "stall_selected", "stall_short_sb", "stall_mio", "stall_barrier"]
agg = collections.defaultdict(lambda: [0.0] * (len(st) + 1))
tot = 0.0
for r in uniq:
    m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)", r[1])
    op = ".".join((m.group(2) if m else "?").split(".")[:2])
    for i, c in enumerate(st):
        agg[op][i] += f(r, c)
    agg[op][-1] += f(r, "Instructions Executed")
    tot += sum(f(r, c) for c in st)
ti = sum(v[-1] for v in agg.values())
print("% of stall samples by reason:",
      {c[6:]: round(100 * sum(v[i] for v in agg.values()) / tot, 1) for i, c in enumerate(st)})
print("opcode".ljust(18), " ".join(c[6:13].rjust(8) for c in st), "  % of instructions")
for op, v in sorted(agg.items(), key=lambda kv: -sum(kv[1][:-1]))[:top]:
    print(op.ljust(18), " ".join(f"{100 * x / tot:8.2f}" for x in v[:-1]), f"{100 * v[-1] / ti:8.2f}")
