set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g8_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g8_pytest.log
timeout 900 python bench.py > gpurun_out/g8_bench.json 2> gpurun_out/g8_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/g8_bench.err
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation"
timeout 300 $B --validation fused > gpurun_out/g8_fused.json 2> gpurun_out/g8_fused.err; echo "fused rc=$?"
timeout 300 $B --validation fused --fps 1000 > gpurun_out/g8_fused1000.json 2> gpurun_out/g8_fused1000.err; echo "f1000 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g8_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing > gpurun_out/g8_ncu.log 2>&1; echo "ncu rc=$?"
