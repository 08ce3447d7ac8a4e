"""Per-CUDA-source-line totals of an ncu report (warp stall samples and warp
instructions executed), from the cuda,sass source page.
usage: ncu_lines.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, lines, tot_s, tot_i = None, [], 0.0, 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        s, i = float(r[4]), float(r[7])
    except (ValueError, IndexError):
        continue
    tot_s += s
    tot_i += i
    lines.append((s, i, f"{fname}:{r[0]}", r[1].strip()))
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
for s, i, loc, src in sorted(lines, reverse=True)[:ntop]:
    print(f"{s / tot_s * 100:5.1f}% stall {i / tot_i * 100:5.1f}% inst  {loc:22s} {src[:80]}")
