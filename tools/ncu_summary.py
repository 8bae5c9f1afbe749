"""Summarise an ncu report: key throughput metrics + top stall sites.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [n_top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread"]
idx = [hdr.index(w) for w in want if w in hdr]
for r in rows[2:]:
    for i in idx:
        print(f"  {hdr[i]:70s} {r[i]} {rows[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    hdr = rows[1]
    data = rows[2:]
    i_src = hdr.index("Source")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in data) or 1
    print(f"  stall samples: {tot:.0f}")
    for k in sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:ntop]:
        r = data[k]
        print(f"  {k:5d} {float(r[i_s] or 0) / tot * 100:5.1f}% ex={r[i_ex]:>9} {r[i_src][:80]}")
