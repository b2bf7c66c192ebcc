#!/bin/bash
# one full ncu capture (with source) of a kernel of the default c4 step:  K=esi_integrate_kernel bash tools/ncu_k2.sh
mkdir -p gpurun_out
K=${K:-esi_integrate_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-20} -c 1 -o gpurun_out/prof_$K -f \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation ${BENCH_ARGS} > gpurun_out/ncu_$K.log 2>&1
echo "ncu $K rc=$?"; tail -3 gpurun_out/ncu_$K.log
