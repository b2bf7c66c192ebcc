#!/bin/bash
# serialized step + launch list + full ncu of K2 (and K1)
mkdir -p gpurun_out
ESI_SINGLE_STREAM=1 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --no-latency --no-alt-validation --steps 5 > gpurun_out/bench_ss.json 2> gpurun_out/bench_ss.err; echo "bench ss rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_ss.json').read().strip().splitlines()[-1]); print('single-stream ms', d['ms_per_step'], d['step_roofline']['kernel_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv 2>&1 | tail -12
for K in ${NCU_K:-esi_integrate_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing > gpurun_out/ncu_$K.log 2>&1; echo "ncu $K rc=$?"
done
