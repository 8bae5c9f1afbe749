"""Per-launch kernel name + duration (+ other metrics) from an ncu --csv log."""
import csv
import sys

rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
d = {}
for r in csv.DictReader(rows):
    d.setdefault(int(r["ID"]), [r["Kernel Name"].split("(")[0][-40:], {}])[1][r["Metric Name"]] = r["Metric Value"]
for i, (n, m) in sorted(d.items()):
    t = float(m.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e3
    extra = " ".join(f"{k.split('__')[-1]}={v}" for k, v in m.items() if k != "gpu__time_duration.sum")
    print(f"{i:3d} {n:40s} {t:8.2f} us  {extra}")
