#!/bin/bash
# A/B of the two band layouts (ESI_BAND_LAYOUT: 0 contiguous, 1 interleaved) on the c4 step,
# on c4 at 1000 FPS, and on locally active scenes (--roi): a centred quarter and a corner sixteenth
mkdir -p gpurun_out
ARGS="--no-cpu-baseline --e2e-steps 0 --no-latency --no-alt-validation --steps 10"
run() {  # name layout extra-args
  ESI_BAND_LAYOUT=$2 timeout 300 python bench.py $ARGS $3 > gpurun_out/abl_$1_$2.json 2> gpurun_out/abl_$1_$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/abl_$1_$2.json').read().strip().splitlines()[-1]); k=d['step_roofline']['kernel_ms_per_step']
print('%-8s layout %s  ms %.3f  %.1f G ev/s  K1 %.3f K2 %.3f  K2 launch %.1f us' % ('$1', '$2', d['ms_per_step'], d['value'] / 1e9, k['esi_partition_kernel'], k['esi_integrate_kernel'], 1e3*d['roofline']['mean_launch_ms']))" || tail -3 gpurun_out/abl_$1_$2.err
}
for rep in 1 2; do
for L in ${LAYOUTS:-0 1}; do
  run c4 $L ""
  run c4k $L "--fps 1000"
  run quarter $L "--roi 0.25,0.25,0.75,0.75"
  run corner $L "--roi 0,0,0.25,0.25"
  run strip $L "--roi 0,0.4,1,0.6"
done
done
