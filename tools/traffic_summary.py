"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) per kernel and write profiles/ncu_traffic.json, which
bench.py reads for roofline.traffic (DRAM bytes per launch of the dominant kernel).

usage: traffic_summary.py gpurun_out/traffic.csv "description of the run" [out.json]"""

import collections
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}

src, desc = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "profiles", "ncu_traffic.json")
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
hdr = rows[0]
ik, im, iv, iu, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per, names = collections.defaultdict(dict), {}
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    per[r[iid]][r[im]] = v * UNITS.get(r[iu], 1.0)
    names[r[iid]] = r[ik].split("(")[0].split("<")[0].replace("void ", "").replace("fr::", "").strip()
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':24s} {'launches':>8s} {'time ms':>10s} {'share':>6s} {'GB/launch':>10s} {'GB/s':>7s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{k:24s} {a[0]:8d} {a[1] * 1e3:10.2f} {a[1] / tot * 100:5.1f}% {a[2] / a[0] / 1e9:10.3f} "
          f"{a[2] / a[1] / 1e9 if a[1] else 0:7.0f}")
res = {}
for k in ("k_sweep", "k_sweep_own", "k_push_block", "k_fold"):
    if k in agg:
        a = agg[k]
        res[k] = round(a[2] / a[0])
        res[k + "_avg_ms_under_ncu"] = round(a[1] / a[0] * 1e3, 4)
        res[k + "_dram_gbs_under_ncu"] = round(a[2] / a[1] / 1e9) if a[1] else None
        res[k + "_launches"] = a[0]
res["source"] = desc
res["round"] = 2
res["kernel_path"] = sys.argv[4] if len(sys.argv) > 4 else "owned"
json.dump(res, open(out, "w"), indent=1)
print("wrote", out)
