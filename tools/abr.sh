#!/bin/bash
# K1 rank modes on the c4 step:  MODES="atomic match peers" bash tools/abr.sh
ARGS="--no-cpu-baseline --e2e-steps 0 --no-latency --no-alt-validation --steps 10"
for rep in 1 2; do
for M in ${MODES:-atomic match}; do
  ESI_RANK_MODE=$M timeout 300 python bench.py $ARGS > gpurun_out/abr_$M.json 2>/dev/null
  ESI_SINGLE_STREAM=1 ESI_RANK_MODE=$M timeout 300 python bench.py $ARGS > gpurun_out/abr_${M}_ss.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/abr_$M.json').read().strip().splitlines()[-1]); s=json.loads(open('gpurun_out/abr_${M}_ss.json').read().strip().splitlines()[-1])
print('%-7s step %.3f ms   serialised %.3f ms  K1 %.3f ms' % ('$M', d['ms_per_step'], s['ms_per_step'], s['step_roofline']['kernel_ms_per_step']['esi_partition_kernel']))"
done
done
