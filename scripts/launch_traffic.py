"""Per-kernel average duration and DRAM traffic per launch from an ncu launch list
(scripts/ncu_capture.sh) -> JSON that bench.py reports as roofline.traffic.

    python scripts/launch_traffic.py gpurun_out/launches_x.csv profiles/traffic_c2.json
"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = {}
for r in rows[h + 1:]:
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("vp::", "")
    d = per.setdefault(name, {}).setdefault(r[ui], {})
    d[r[mi]] = float(r[vi].replace(",", ""))
out = {}
for name, launches in per.items():
    n = len(launches)
    tot = lambda m: sum(v.get(m, 0.0) for v in launches.values())  # noqa: E731
    out[name] = {"launches": n, "avg_us": tot("gpu__time_duration.sum") / n / 1e3,
                 "dram_bytes_per_launch": (tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum")) / n}
json.dump({"source": sys.argv[1], "kernels": out}, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
