mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g25_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g25_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation"
timeout 300 $B > gpurun_out/g25_push.json 2> gpurun_out/g25_push.err; echo "push rc=$?"
python - gpurun_out/g25_push.json <<'PY'
import json,sys
for l in open(sys.argv[1]):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['value']/1e9,2), 'G ev/s', round(d['ms_per_step'],3),'ms', {k:round(v,3) for k,v in d['step_roofline']['kernel_ms_per_step'].items()})
PY
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing"
timeout 900 ncu --set full --clock-control none -k regex:esi_validate -s 1 -c 1 -o gpurun_out/ncu_val2 -f $CMD > gpurun_out/ncu_val2.log 2>&1; echo "ncu rc=$?"
