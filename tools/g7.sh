set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/g7_bench.err
timeout 600 python bench.py --config c5b --steps 3 --warmup 1 > gpurun_out/g7_c5b.json 2> gpurun_out/g7_c5b.err; echo "c5b rc=$?"
tail -3 gpurun_out/g7_c5b.err
timeout 300 python -m pytest tests/test_esim.py -q -m gpu > gpurun_out/g7_esim.log 2>&1; tail -3 gpurun_out/g7_esim.log
