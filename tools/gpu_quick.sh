#!/bin/bash
# parity tests + bench (+ optional ncu launch list)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value %.4g ev/s  ms/step %.3f  frames/s %.4g" % (d["value"], d["ms_per_step"], d["frames_per_s"]))
    print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac", "mean_launch_ms")})
    print("step", d["step_roofline"])
    print("e2e", d.get("e2e")); print("clocks", d.get("clocks"))
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.err").read()[-3000:])
PY
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
  for K in $NCU; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$K.log 2>&1; echo "ncu $K rc=$?"
  done
fi
