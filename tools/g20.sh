mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_slice_maps.py -m gpu -q -x > gpurun_out/g20_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g20_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation"
timeout 300 $B > gpurun_out/g20_push.json 2> gpurun_out/g20_push.err; echo "push rc=$?"
timeout 300 $B --validation fused > gpurun_out/g20_fused.json 2> gpurun_out/g20_fused.err; echo "fused rc=$?"
timeout 300 $B --validation fused --fps 1000 > gpurun_out/g20_f1000.json 2> gpurun_out/g20_f1000.err; echo "f1000 rc=$?"
for f in gpurun_out/g20_*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['value']/1e9,2), 'G ev/s', round(d['ms_per_step'],3),'ms', {k:round(v,3) for k,v in d['step_roofline']['kernel_ms_per_step'].items()})
PY
done
