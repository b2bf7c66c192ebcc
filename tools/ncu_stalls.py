"""Stall reasons per source line (and totals) of one kernel in an ncu report.

    python tools/ncu_stalls.py report.ncu-rep [top_n]
"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None; cur = ""; tot = collections.Counter(); per = collections.defaultdict(collections.Counter); src = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or not r[0].isdigit():
        continue
    key = f"{cur}:{r[0]}"
    src[key] = r[1].strip()[:70]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = float(r[i] or 0)
            except ValueError:
                continue
            tot[h] += v; per[key][h] += v
T = sum(tot.values()) or 1
print("totals:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in tot.most_common(10)))
for key, c in sorted(per.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(c.values())
    print(f"{key:28s} {100*s/T:5.1f}%  " + " ".join(f"{k[6:]}:{100*v/T:.1f}" for k, v in c.most_common(3)) + "  | " + src[key])
