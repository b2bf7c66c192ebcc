"""Per-line instruction counts / stall samples of an ncu report (CUDA source view),
optionally summed over line ranges:  python tools/ncu_lines.py rep file.cu a-b:name ..."""
import csv, io, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = ""; hdr = None; per = {}
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": cur = row[1].split("/")[-1]; continue
    if row[0] == "Line No":
        hdr = row; wi = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed"); continue
    if hdr is None or row[0] in ("", "Function Name"): continue
    try: ln = int(row[0])
    except ValueError: continue
    k = (cur, ln)
    a, b = per.get(k, (0, 0))
    try:
        per[k] = (a + int(row[ii] or 0), b + int(row[wi] or 0))
    except (ValueError, IndexError):
        pass
tot_i = sum(v[0] for v in per.values()); tot_s = sum(v[1] for v in per.values())
print("total inst", tot_i, "samples", tot_s)
acc = 0
for spec in sys.argv[3:]:
    rng, name = spec.split(":")
    a, b = map(int, rng.split("-"))
    i = sum(v[0] for (f, l), v in per.items() if f == fname and a <= l <= b)
    s = sum(v[1] for (f, l), v in per.items() if f == fname and a <= l <= b)
    acc += i
    print(f"{name:12s} lines {a}-{b}: inst {i/1e6:7.1f} M ({100*i/tot_i:4.1f}%)  samples {100*s/tot_s:4.1f}%")
others = {f: 0 for f, _ in per}
for (f, l), v in per.items():
    if f != fname: others[f] += v[0]
for f, v in others.items():
    if v: print(f"{f:30s} inst {v/1e6:7.1f} M")
