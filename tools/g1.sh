set -x
mkdir -p gpurun_out
./tools/micro/rank > gpurun_out/micro_rank.txt 2>&1
./tools/micro/micro > gpurun_out/micro_base.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_r02_base.json 2> gpurun_out/bench_r02_base.err
echo done
