"""Summarise an ncu report: headline metrics, stall reasons and the top
stalled SASS lines.  usage: ncu_summary.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 14
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__bytes.sum.per_second',
        'lts__t_sectors_srcunit_tex_op_red.sum', 'sm__warps_active.avg.pct', 'lts__throughput.avg.pct',
        'l1tex__throughput.avg.pct', 'smsp__issue_active.avg.pct', 'smsp__inst_executed.sum',
        'launch__registers_per_thread']
for d in data:
    for i, h in enumerate(hdr):
        if any(p in h for p in keys) or ('pcsamp_warps_issue_stalled' in h and 'not_issued' not in h):
            try:
                v = float(d[i])
            except ValueError:
                continue
            if v == 0 or ('pcsamp' in h and v < 1500):
                continue
            print(f'  {h} [{units[i]}] = {d[i]}')
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
isrc = hdr.index('Source'); iws = hdr.index('Warp Stall Sampling (All Samples)'); iie = hdr.index('Instructions Executed')
lst, tot = [], 0.0
for k, r in enumerate(data):
    try:
        ws = float(r[iws]); ie = float(r[iie])
    except ValueError:
        continue
    tot += ws
    lst.append((ws, ie, k, r[isrc].strip()))
for ws, ie, k, s in sorted(lst, reverse=True)[:ntop]:
    print(f'{ws / tot * 100:5.1f}% stall  [{k}] x{ie:.0f} {s[:90]}')
