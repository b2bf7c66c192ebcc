"""Summarise an ncu report's source page: CUDA lines ranked by warp-stall samples.

    python tools/ncu_hot.py report.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file = ""
res = []
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or row[0] in ("", "Function Name"):
        continue
    try:
        res.append((float(row[wi]), row[ii], cur_file, row[0], row[1]))
    except (ValueError, IndexError):
        pass
tot = sum(r[0] for r in res) or 1
print(f"total stall samples {tot:.0f}")
for s, inst, f, ln, src in sorted(res, key=lambda r: -r[0])[:n]:
    print(f"{s:8.0f} {100 * s / tot:5.1f}%  inst {inst:>9s}  {f}:{ln:<5s} {src.strip()[:100]}")
