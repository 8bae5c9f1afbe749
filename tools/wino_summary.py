"""Winograd transform kernels' HBM fraction from an ncu launch list of
tools/wino_probe.py (metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum, dram__throughput.avg.pct_of_peak_sustained_elapsed):
    python tools/wino_summary.py launches.csv [layer]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                   hdr.index("ID"))
launch = {}
for r in rows[1:]:
    d = launch.setdefault(int(r[iid]), {"kernel": r[ik]})
    d[r[im]] = float(r[iv].replace(",", ""))
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''} Winograd kernels (ncu, cold L2): time, DRAM bytes, "
      "achieved GB/s, dram__throughput % of peak")
for i in sorted(launch):
    d = launch[i]
    k = d["kernel"].split("(")[0].replace("void ", "").replace("tkb::<unnamed>::", "")
    if not any(x in k for x in ("wino", "tc_gemm", "exact_gemm", "split3")):
        continue
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{k[:58]:58s} {t:8.1f} us {b:8.1f} MB {b / max(t, 1e-9) * 1e3:7.0f} GB/s "
          f"{d.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%")
