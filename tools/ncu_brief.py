"""Brief per-kernel digest of an ncu --set full report (development aid):
python tools/ncu_brief.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
WANT = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
stalls = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and
          c.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:80])
    for w in WANT:
        if w in h:
            print(f"   {w:75s} {r[h.index(w)]}")
    st = sorted(((float(r[h.index(c)] or 0), c) for c in stalls), reverse=True)[:9]
    print("   stalls/issue:", ", ".join(f"{c[34:-27]} {v:.2f}" for v, c in st))
