#!/bin/bash
# A/B of libesi variants on the c4 step (and optionally 1000 FPS / c3):  LIBS="old cur" bash tools/ab.sh
mkdir -p gpurun_out
ARGS="--no-cpu-baseline --e2e-steps 0 --no-latency --no-alt-validation --steps 10"
for rep in 1 2; do
for L in ${LIBS:-old cur}; do
  if [ "$L" = cur ]; then P=paper_2508_02238_b200/libesi.so; else P=paper_2508_02238_b200/variants/libesi_$L.so; fi
  for FPS in ${FPSS:-100}; do
    ESI_LIB_PATH=$P timeout 300 python bench.py $ARGS --fps $FPS > gpurun_out/ab_${L}_${FPS}.json 2> gpurun_out/ab_${L}_${FPS}.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_${L}_${FPS}.json').read().strip().splitlines()[-1]); k=d['step_roofline']['kernel_ms_per_step']
print('%-10s fps %5s  ms %.3f  K1 %.3f K2 %.3f  K2 launch %.1f us' % ('$L', '$FPS', d['ms_per_step'], k['esi_partition_kernel'], k['esi_integrate_kernel'], 1e3*d['roofline']['mean_launch_ms']))" || tail -3 gpurun_out/ab_${L}_${FPS}.err
  done
  if [ -n "$SS" ]; then
    ESI_SINGLE_STREAM=1 ESI_LIB_PATH=$P timeout 300 python bench.py $ARGS > gpurun_out/ab_${L}_ss.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab_${L}_ss.json').read().strip().splitlines()[-1]); k=d['step_roofline']['kernel_ms_per_step']
print('%-10s single-stream ms %.3f  K1 %.3f K2 %.3f' % ('$L', d['ms_per_step'], k['esi_partition_kernel'], k['esi_integrate_kernel']))"
  fi
done
done
