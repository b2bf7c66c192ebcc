mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for L in libesi.so libesi_k3.so libesi.so libesi_k3.so; do
  echo "== $L"; ESI_LIB_PATH=$PWD/paper_2508_02238_b200/$L timeout 600 python tools/bench_configs.py c3 c4 c4@1000 2>&1 | tail -3
done
