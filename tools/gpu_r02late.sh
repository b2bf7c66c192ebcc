#!/bin/bash
# Late round-2 measurement set -> gpurun_out/ (copied to profiles/r02_late/)
bash tools/gpu_final.sh
timeout 600 python bench.py --config c5a --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c5a.json 2> gpurun_out/bench_c5a.err; echo "c5a rc=$?"
timeout 600 python bench.py --config c5b --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err; echo "c5b rc=$?"
timeout 600 python bench.py --config c4t --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c4t.json 2> gpurun_out/bench_c4t.err; echo "c4t rc=$?"
timeout 600 python tools/bench_slices.py > gpurun_out/slices.json 2> gpurun_out/slices.err; echo "slices rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_validate -s 1 -c 1 -o gpurun_out/prof_esi_validate -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing > gpurun_out/ncu_validate.log 2>&1; echo "ncu validate rc=$?"
