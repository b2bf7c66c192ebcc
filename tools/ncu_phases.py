"""Per-source-line instruction counts and stall samples of one kernel in an ncu report.

    python tools/ncu_phases.py report.ncu-rep file.cu [top_n]
"""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, cur, res = None, "", []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].isdigit() or cur != fname:
        continue
    try:
        res.append((int(r[0]), float(r[ii] or 0), float(r[si] or 0), r[1].strip()[:90]))
    except ValueError:
        pass
ti = sum(x[1] for x in res) or 1
ts = sum(x[2] for x in res) or 1
print(f"{fname}: {ti:.0f} warp instructions, {ts:.0f} stall samples")
for l, v, st, src in sorted(res, key=lambda x: -x[1])[:n]:
    print(f"{l:5d} inst {v:10.0f} {100 * v / ti:5.1f}%  stall {100 * st / ts:5.1f}%  {src}")
