#!/bin/bash
# parity suite + bench on the current build
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value %.4g ev/s  ms/step %.3f" % (d["value"], d["ms_per_step"]), d["step_roofline"]["kernel_ms_per_step"], d.get("other_validation_mode", {}).get("ms_per_step"))
    print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac", "mean_launch_ms")})
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.err").read()[-3000:])
PY
