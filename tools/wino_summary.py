"""Winograd transform kernels' HBM fraction from an ncu launch list of
tools/wino_probe.py (metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum, dram__throughput.avg.pct_of_peak_sustained_elapsed):
    python tools/wino_summary.py launches.csv layer
For the transforms it also prints the ALGORITHMIC bytes (input
transform reads 4 N H W C and writes 4 T^2 tiles C; output transform reads
4 T^2 tiles K and writes 4 N OH OW K) over the kernel time, against the
measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs) -- ncu's DRAM counter
misses the transform-domain writes still in L2 when the kernel ends."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                   hdr.index("ID"))
launch = {}
for r in rows[1:]:
    d = launch.setdefault(int(r[iid]), {"kernel": r[ik]})
    d[r[im]] = float(r[iv].replace(",", ""))
from bench import VGG16  # noqa: E402
layer = sys.argv[2]
h, c, kf = [(hh, cc, kk) for n, hh, cc, kk, _ in VGG16 if n == layer][0]
try:
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except OSError:
    hbm = 6535.4


def algo_bytes(kname):
    m = 2 if "F2" in kname else 4
    t = m + 2
    tiles = 32 * ((h + m - 1) // m) ** 2
    if "wino_input" in kname:
        return 4 * 32 * h * h * c + 4 * t * t * tiles * c
    if "wino_output" in kname:
        return 4 * t * t * tiles * kf + 4 * 32 * h * h * kf
    return None


print(f"# {layer} (batch 32) Winograd kernels, ncu cold L2: time, DRAM bytes, DRAM GB/s, "
      f"dram__throughput %; transforms: algorithmic bytes, GB/s, % of the {hbm:.0f} GB/s copy peak")
for i in sorted(launch):
    d = launch[i]
    k = d["kernel"].split("(")[0].replace("void ", "").replace("tkb::<unnamed>::", "")
    if not any(x in k for x in ("wino", "tc_gemm", "exact_gemm", "split3")):
        continue
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    line = (f"{k[:44]:44s} {t:7.1f} us {b:7.1f} MB {b / max(t, 1e-9) * 1e3:6.0f} GB/s "
            f"{d.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%")
    ab = algo_bytes(k)
    if ab:
        gbs = ab / 1e6 / max(t, 1e-9) * 1e3
        line += f" | algorithmic {ab / 1e6:7.1f} MB {gbs:6.0f} GB/s {100 * gbs / hbm:5.1f}%"
    print(line)
