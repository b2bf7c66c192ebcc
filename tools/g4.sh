set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g4_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g4_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency"
timeout 300 $B > gpurun_out/g4_w2.json 2> gpurun_out/g4_w2.err; echo "w2 rc=$?"
timeout 300 $B --fps 1000 --no-alt-validation > gpurun_out/g4_w2_1000.json 2> gpurun_out/g4_w2_1000.err
for f in gpurun_out/g4_*.json; do echo $f; python -c "
import json,sys
for l in open('$f'):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(' ', d.get('value'), d.get('ms_per_step'), d.get('step_roofline',{}).get('kernel_ms_per_step'), d.get('other_validation_mode'))
"; done
CMD="python bench.py --steps 1 --warmup 2 --e2e-steps 0 --no-cpu-baseline --no-kernel-timing --no-latency --no-alt-validation"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_integrate_w2 -s 30 -c 1 -o gpurun_out/prof_w21 -f $CMD > gpurun_out/ncu_w21.log 2>&1; echo "ncu rc=$?"
