#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list, ncu full captures of K1/K2.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_partition -s 20 -c 1 -o gpurun_out/prof_part -f $CMD > gpurun_out/ncu_part.log 2>&1; echo "ncu part rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_integrate -s 20 -c 1 -o gpurun_out/prof_int -f $CMD > gpurun_out/ncu_int.log 2>&1; echo "ncu int rc=$?"
