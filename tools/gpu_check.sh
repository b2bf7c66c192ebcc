#!/bin/bash
# GPU suite (normal + checked build), router throughput, one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
ESI_LIB_PATH=$PWD/paper_2508_02238_b200/libesi_checked.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_checked.log 2>&1; echo "checked rc=$?"; tail -2 gpurun_out/pytest_checked.log
timeout 300 python tools/bench_route.py > gpurun_out/route.json 2>&1; echo "route rc=$?"; tail -2 gpurun_out/route.json
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.json
