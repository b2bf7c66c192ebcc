mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation"
for v in default overlap overlap4k; do
  if [ $v = default ]; then L=""; else L="ESI_LIB_PATH=paper_2508_02238_b200/variants/libesi_$v.so"; fi
  env $L timeout 300 $B --validation fused > gpurun_out/g22_${v}_fused.json 2> gpurun_out/g22_$v.err; echo "$v rc=$?"
  env $L timeout 300 $B > gpurun_out/g22_${v}_push.json 2>> gpurun_out/g22_$v.err
  env $L timeout 300 $B --validation fused --fps 1000 > gpurun_out/g22_${v}_f1000.json 2>> gpurun_out/g22_$v.err
  env $L ESI_SINGLE_STREAM=1 timeout 300 $B --validation fused > gpurun_out/g22_${v}_serial.json 2>> gpurun_out/g22_$v.err
done
for f in gpurun_out/g22_*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['value']/1e9,2), 'G ev/s', round(d['ms_per_step'],3),'ms', {k:round(v,3) for k,v in d['step_roofline']['kernel_ms_per_step'].items()})
PY
done
