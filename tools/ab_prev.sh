#!/bin/bash
# previous build (variants/libesi_prev.so) vs the current one: c4 @100 / @1000 FPS, c3, both layouts at 100 FPS
mkdir -p gpurun_out
ARGS="--no-cpu-baseline --e2e-steps 0 --no-latency --no-alt-validation --steps 10"
run() {  # name lib layout extra-args
  ESI_LIB_PATH=$2 ESI_BAND_LAYOUT=$3 timeout 300 python bench.py $ARGS $4 > gpurun_out/abp_$1.json 2> gpurun_out/abp_$1.err
  python -c "
import json; d=json.loads(open('gpurun_out/abp_$1.json').read().strip().splitlines()[-1]); k=d['step_roofline']['kernel_ms_per_step']
print('%-12s ms %.3f  %.1f G ev/s  K1 %.3f K2 %.3f  K2 launch %.1f us' % ('$1', d['ms_per_step'], d['value'] / 1e9, k['esi_partition_kernel'], k['esi_integrate_kernel'], 1e3*d['roofline']['mean_launch_ms']))" || tail -3 gpurun_out/abp_$1.err
}
PREV=paper_2508_02238_b200/variants/libesi_prev.so
CUR=paper_2508_02238_b200/libesi.so
for rep in 1 2; do
  run prev100 $PREV 0 ""
  run cur100 $CUR 0 ""
  run prev1000 $PREV 0 "--fps 1000"
  run cur1000 $CUR 0 "--fps 1000"
  run prev100il $PREV 1 ""
  run cur100il $CUR 1 ""
done
