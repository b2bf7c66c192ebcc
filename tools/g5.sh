set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g5_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g5_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency"
for K2 in block warp; do
for RM in peers atomic ballot; do
ESI_K2=$K2 ESI_RANK_MODE=$RM timeout 300 $B > gpurun_out/g5_${K2}_${RM}.json 2> gpurun_out/g5_${K2}_${RM}.err
done; done
for f in gpurun_out/g5_*.json; do echo $f; python -c "
import json,sys
for l in open('$f'):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(' ', round(d.get('ms_per_step'),3), {k:round(v,3) for k,v in d.get('step_roofline',{}).get('kernel_ms_per_step').items()}, round(d.get('other_validation_mode',{}).get('ms_per_step',0),3))
"; done
