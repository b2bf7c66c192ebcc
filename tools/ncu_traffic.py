"""Per-launch DRAM traffic of the kernels in ncu --set full reports -> profiles/traffic.json.

    python tools/ncu_traffic.py out.json report1.ncu-rep [report2.ncu-rep ...]

traffic = dram__bytes_read.sum + dram__bytes_write.sum of the captured launch
(bench.py reads it for its roofline "traffic" field).
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "lts__t_bytes.sum"):
            if k in hdr:
                i = hdr.index(k)
                v = r[i]
                if k != "Kernel Name":
                    v = float(v.replace(",", "")) * UNITS.get(units[i], 1.0 if units[i] != "usecond" else 1.0)
                d[k] = v
        res.append(d)
    return res


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    try:
        data = json.load(open(out))
    except Exception:
        data = {}
    for rep in reps:
        for d in metrics(rep):
            name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1].strip()
            data[name] = {"dram_bytes_per_launch": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
                          "dram_read": d.get("dram__bytes_read.sum"), "dram_write": d.get("dram__bytes_write.sum"),
                          "l2_bytes": d.get("lts__t_bytes.sum"), "duration_us": d.get("gpu__time_duration.sum"),
                          "source": rep.split("/")[-1]}
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
