"""Condense an ncu --csv launch list (gpu__time_duration + dram bytes) into
per-kernel shares of the timed step.  Usage: launch_summary.py launches.csv out.json"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                   hdr.index("ID"))
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[iid], {"kernel": r[ik]})
    d[r[im]] = float(r[iv].replace(",", ""))
ls = list(launch.values())
# The timed step = every launch after the last L2-flush fill kernel.
last_fill = max(i for i, d in enumerate(ls) if "FillFunctor" in d["kernel"])
step = ls[last_fill + 1:]
total = sum(d.get("gpu__time_duration.sum", 0) for d in step)
agg = collections.OrderedDict()
for d in step:
    name = d["kernel"].split("(")[0].replace("void ", "")
    a = agg.setdefault(name, {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0})
    a["launches"] += 1
    a["time_ns"] += d.get("gpu__time_duration.sum", 0)
    a["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
for a in agg.values():
    a["share"] = round(a["time_ns"] / total, 4)
out = {"source": sys.argv[1], "launches_in_window": len(step), "window_time_ns": total,
       "kernels": agg,
       "per_launch": [{"kernel": d["kernel"][:90], "ns": d.get("gpu__time_duration.sum"),
                       "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)}
                      for d in step]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, a in agg.items():
    print(f"{a['share']*100:5.1f}%  n={a['launches']:3d}  {a['time_ns']/1e3:9.1f} us  dram={a['dram_bytes']/1e6:9.1f} MB  {k[:70]}")
