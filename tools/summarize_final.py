"""Copy one `tools/gpu_final.sh` run from gpurun_out/ into profiles/<name>/ and
write its SUMMARY.md (bench lines, ncu launch list, ncu kernel details, per
config table, router, tests).

    python tools/summarize_final.py [name] [build-note]
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out")
NAME = sys.argv[1] if len(sys.argv) > 1 else "r01_final"
NOTE = sys.argv[2] if len(sys.argv) > 2 else ""
DST = os.path.join(ROOT, "profiles", NAME)


def last_json(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def tail(path, n=1):
    with open(path) as f:
        return f.read().strip().splitlines()[-n:]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if not r:
            continue
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("esi::", "")
        name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v *= {"usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    return ["| `%s` | %d | %.1f | %.2f | %.1f %% |" % (k, n, t / 1e3, t / n / 1e3, 100 * t / tot)
            for k, (n, t) in agg.items()]


def ncu_metric(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    res, hdr = {}, None
    for r in csv.reader(out.splitlines()):
        if "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) >= hdr.index("Metric Value") + 1:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") in names:
                res[d["Metric Name"]] = (d.get("Metric Value"), d.get("Metric Unit"))
    return res


def main():
    os.makedirs(DST, exist_ok=True)
    for f in ("bench.json", "bench_1000fps.json", "bench_ref.json", "configs.jsonl", "launches.csv", "lscpu.txt",
              "nvsmi.txt", "pytest_gpu.log", "pytest_checked.log", "smoke.log", "traffic.json"):
        if os.path.exists(os.path.join(SRC, f)):
            shutil.copy(os.path.join(SRC, f), DST)
    if os.path.exists(os.path.join(SRC, "route_1.json")):
        shutil.copy(os.path.join(SRC, "route_1.json"), os.path.join(DST, "route.json"))
    if os.path.exists(os.path.join(SRC, "traffic.json")):
        shutil.copy(os.path.join(SRC, "traffic.json"), os.path.join(ROOT, "profiles", "traffic.json"))
    det = {}
    for k in ("esi_partition", "esi_integrate"):
        rep = os.path.join(SRC, f"prof_{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        with open(os.path.join(DST, f"ncu_{k}_details.csv"), "w") as f:
            f.write(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                                   text=True).stdout)
        with open(os.path.join(DST, f"ncu_{k}_lines.txt"), "w") as f:
            f.write(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "40"],
                                   capture_output=True, text=True).stdout)
        det[k] = ncu_metric(rep, {"Duration", "DRAM Throughput", "Executed Ipc Active", "Achieved Occupancy"})

    b = last_json(os.path.join(DST, "bench.json"))
    f1k = last_json(os.path.join(DST, "bench_1000fps.json"))
    ref = last_json(os.path.join(DST, "bench_ref.json"))
    rf, sr, e2e, clk = b["roofline"], b["step_roofline"], b["e2e"], b["clocks"]
    tr = json.load(open(os.path.join(DST, "traffic.json")))
    L = ["# Round 1 — final measurements (B200, 1 GPU)", "",
         "Commands: `bash tools/gpu_final.sh` (= `tools/gpu_all.sh` + router + per-config benches + "
         "checked-build tests); summary by `python tools/summarize_final.py`.", ""]
    if NOTE:
        L += [NOTE, ""]
    L += ["## bench.py (c4: 1280x720, %d events, 1000 frames @100 FPS)" % b["config"]["events_per_step_per_gpu"], "",
          "* value **%.2f G events/s**, %.3f ms/step, %.0f frames/s, clocks %s/%s MHz, reasons %s"
          % (b["value"] / 1e9, b["ms_per_step"], b["frames_per_s"], clk["sm_mhz"], clk["sm_max_mhz"], clk["reasons"]),
          "* roofline (dominant kernel `%s`): achieved %.0f GB/s of %.1f GB/s = %.1f %%; ncu traffic %.1f MB/launch"
          % (rf["kernel"], rf["achieved"], rf["peak"], 100 * rf["frac"], (rf["traffic"] or 0) / 1e6),
          "  (its algorithmic bytes are only the frames + state; it is bound by the per-window latency chain, "
          "DESIGN.md 4)",
          "* step-level: %.2f GB algorithmic per step -> %.0f GB/s = %.1f %% of HBM"
          % (sr["algorithmic_bytes"] / 1e9, sr["achieved_gbs"], 100 * sr["frac"]),
          "* e2e (C ABI with pinned host buffers, pipelined copies): %.2f G events/s (%.1f ms/step; PCIe-bound: "
          "%.1f GB H2D + %.2f GB D2H per step)" % (e2e["value"] / 1e9, e2e["ms_per_step"],
                                                   e2e["h2d_bytes_per_step"] / 1e9, e2e["d2h_bytes_per_step"] / 1e9),
          "* cpu_baseline (fp64 oracle, %d core): %.2f M events/s; `--impl reference`: %.2f M events/s"
          % (b["cpu_baseline"]["cores"], b["cpu_baseline"]["value"] / 1e6, ref["value"] / 1e6),
          "* 1000 FPS: **%.2f G events/s**, %.2f ms/step, %.0f frames/s" % (f1k["value"] / 1e9, f1k["ms_per_step"],
                                                                          f1k["frames_per_s"]),
          "* gpu_launches %d per timed region (%d steps)" % (b["gpu_launches"], b["steps"]), "",
          "## ncu launch list (`launches.csv`; serialized, cold-cache)", "",
          "| kernel | launches | total µs | mean µs | share |", "|---|---|---|---|---|"]
    L += launch_table(os.path.join(DST, "launches.csv"))
    L += ["", "## ncu --set full, one launch each (`ncu_*_details.csv`, `ncu_*_lines.txt`)", ""]
    for k, name in (("esi_partition", "esi_partition_kernel"), ("esi_integrate", "esi_integrate_kernel")):
        d = det.get(k, {})
        t = tr.get(name, {})
        L.append("* %s: %s µs per chunk; DRAM %.0f MB read + %.0f MB written; DRAM throughput %s %%, IPC %s, "
                 "achieved occupancy %s %%" % (name, d.get("Duration", ("?",))[0], t.get("dram_read", 0) / 1e6,
                                               t.get("dram_write", 0) / 1e6, d.get("DRAM Throughput", ("?",))[0],
                                               d.get("Executed Ipc Active", ("?",))[0],
                                               d.get("Achieved Occupancy", ("?",))[0]))
    L += ["", "## Per config (`configs.jsonl`, device-resident inputs)", "",
          "| config | fps | ms | G events/s | step HBM fraction |", "|---|---|---|---|---|"]
    for line in open(os.path.join(DST, "configs.jsonl")):
        d = json.loads(line)
        L.append("| %s | %d | %.3f | %.2f | %.1f %% |" % (d["config"], d["fps"], d["ms"], d["events_per_s"] / 1e9,
                                                          100 * d["step_hbm_frac"]))
    if os.path.exists(os.path.join(DST, "route.json")):
        r = last_json(os.path.join(DST, "route.json"))
        L += ["", "## Row-band router (`route.json`)", "",
              "%d events of a %s stream into %d bands: %.2f ms/call = %.1f G events/s, %.0f GB/s algorithmic "
              "(48 B/event) = %.0f %% of HBM." % (r["events"], r["sensor"], r["bands"], r.get("ms_per_call", r.get("count_plus_scatter_ms")),
                                                  r["events_per_s"] / 1e9, r["achieved_gbs"], 100 * r["frac"])]
    L += ["", "## Tests", "",
          "`pytest -m gpu`: %s (`pytest_gpu.log`); against the checked build (device invariant traps): %s "
          "(`pytest_checked.log`); `smoke()`: %s" % (tail(os.path.join(DST, "pytest_gpu.log"))[0].strip(),
                                                     tail(os.path.join(DST, "pytest_checked.log"))[0].strip(),
                                                     tail(os.path.join(DST, "smoke.log"))[0].strip())]
    with open(os.path.join(DST, "SUMMARY.md"), "w") as f:
        f.write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
