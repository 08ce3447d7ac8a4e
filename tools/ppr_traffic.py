"""DRAM bytes and L2 reduction sectors of one batched-PPR solve from an ncu
--graph-profiling graph launch list (the solve is one CUDA graph: the last
"graph" entry is the timed solve of tools/ppr_prof.py), written to
profiles/r02_ppr_traffic.json (read by bench.py for ppr.roofline.traffic).
usage: ppr_traffic.py launches.csv "description" [out.json]"""
import csv
import json
import os
import sys

src, desc = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "profiles", "r02_ppr_traffic.json")
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
hdr = rows[0]
ik, im, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
graphs = {}
for r in rows[1:]:
    if r[ik].strip() == "graph":
        graphs.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", ""))
last = graphs[max(graphs, key=int)]
rd, wr = last["dram__bytes_read.sum"], last["dram__bytes_write.sum"]
ms = last["gpu__time_duration.sum"] / 1e6
res = {"source": desc, "solve_ms_under_ncu": round(ms, 3), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
       "dram_bytes_per_solve": int(rd + wr), "dram_tbs_under_ncu": round((rd + wr) / (ms * 1e-3) / 1e12, 3),
       "red_sectors": int(last["lts__t_sectors_srcunit_tex_op_red.sum"]),
       "red_sectors_per_s": round(last["lts__t_sectors_srcunit_tex_op_red.sum"] / (ms * 1e-3) / 1e9, 2)}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
