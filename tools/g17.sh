mkdir -p gpurun_out
timeout 300 python tools/bench_route.py > gpurun_out/g17_route.json 2> gpurun_out/g17_route.err; echo "route rc=$?"; tail -2 gpurun_out/g17_route.err
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation"
for v in default k2c2 k2c2_t2048 t2048c3; do
  if [ $v = default ]; then L=""; else L="ESI_LIB_PATH=paper_2508_02238_b200/variants/libesi_$v.so"; fi
  env $L timeout 300 $B > gpurun_out/g17_$v.json 2> gpurun_out/g17_$v.err; echo "$v rc=$?"
  env $L timeout 300 $B --validation fused > gpurun_out/g17_${v}_fused.json 2>> gpurun_out/g17_$v.err
  env $L timeout 300 $B --validation fused --fps 1000 > gpurun_out/g17_${v}_f1000.json 2>> gpurun_out/g17_$v.err
done
for f in gpurun_out/g17_*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l)
        if 'ms_per_step' in d: print(sys.argv[1], round(d['value']/1e9,2), 'G ev/s', round(d['ms_per_step'],3),'ms', {k:round(v,3) for k,v in d['step_roofline']['kernel_ms_per_step'].items()})
        else: print(sys.argv[1], {k: v for k, v in d.items() if k != 'samples_ms'})
PY
done
