set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g6_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g6_pytest.log
timeout 900 python bench.py > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/g6_bench.err
timeout 600 python bench.py --config c5b --steps 3 --warmup 1 > gpurun_out/g6_c5b.json 2> gpurun_out/g6_c5b.err; echo "c5b rc=$?"
tail -3 gpurun_out/g6_c5b.err
timeout 600 python bench.py --config c5a --steps 2 --warmup 1 > gpurun_out/g6_c5a.json 2> gpurun_out/g6_c5a.err; echo "c5a rc=$?"
tail -3 gpurun_out/g6_c5a.err
