"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    unit = r[ui]
    v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
for k, (n, t) in agg.items():
    print(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f} % |")
