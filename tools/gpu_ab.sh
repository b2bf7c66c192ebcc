#!/bin/bash
# GPU parity tests of the current build, then A/B of libesi variants on the c4 step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
LIBS="${LIBS:-old cur}" FPSS="${FPSS:-100 1000}" bash tools/ab.sh
