"""Per-CUDA-source-line totals of an ncu report (warp stall samples, warp
instructions executed, L1 shared-memory wavefronts and global L1 tag requests),
from the cuda,sass source page.  Lines of inlined helpers are counted both at the
helper's line and at its call site.
usage: ncu_lines.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
COLS = ("Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Ideal", "L1 Tag Requests Global")
fname, hdr, recs = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    try:
        int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr[2:], r[2:]))  # the first two columns are "Line No", "Source"

    def val(k):
        try:
            return float(d.get(k) or 0)
        except ValueError:
            return 0.0
    recs.append(tuple(val(k) for k in COLS) + (f"{fname}:{r[0]}", r[1].strip()))
tot = [sum(x[i] for x in recs) or 1.0 for i in range(len(COLS))]
print(f"total stall samples {tot[0]:.0f}, warp instructions {tot[1]:.3e}, shared wavefronts {tot[2]:.3e} "
      f"(ideal {tot[3]:.3e}), global tag requests {tot[4]:.3e}")
print(" stall%  inst%  shW%  shW/ideal  location               source")
for x in sorted(recs, reverse=True)[:ntop]:
    ratio = f"{x[2] / x[3]:5.1f}x" if x[3] else "   - "
    print(f"{x[0] / tot[0] * 100:6.1f} {x[1] / tot[1] * 100:6.1f} {x[2] / tot[2] * 100:5.1f}  {ratio}     "
          f"{x[5]:22s} {x[6][:70]}")
