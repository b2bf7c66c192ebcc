#!/bin/bash
# default bench line (clock sampling fixed) + clean ncu launch list of the default step
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv
