#!/bin/bash
# baseline re-measure in a fresh container: bench + full ncu captures of K2 and K1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.json
for K in esi_integrate_kernel esi_partition_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$K.log 2>&1; echo "ncu $K rc=$?"
done
