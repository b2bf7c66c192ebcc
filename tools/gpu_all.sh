#!/bin/bash
# Full GPU session: parity tests, bench (100 and 1000 FPS), ncu launch list,
# ncu --set full captures of K1/K2, traffic summary.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --fps 1000 --steps 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_1000fps.json 2> gpurun_out/bench_1000fps.err; echo "bench1000 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
for K in esi_partition esi_integrate; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1; echo "ncu $K rc=$?"
done
python tools/ncu_traffic.py gpurun_out/traffic.json gpurun_out/prof_esi_partition.ncu-rep gpurun_out/prof_esi_integrate.ncu-rep > /dev/null 2>&1
