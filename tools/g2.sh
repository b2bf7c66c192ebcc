set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g2_pytest.log
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/g2_w2.json 2> gpurun_out/g2_w2.err; echo "w2 rc=$?"
timeout 300 $B --fps 1000 > gpurun_out/g2_w2_1000.json 2> gpurun_out/g2_w2_1000.err
ESI_K2_CTAS=1 timeout 300 $B > gpurun_out/g2_w2_c1.json 2>&1
ESI_K2_CTAS=3 timeout 300 $B > gpurun_out/g2_w2_c3.json 2>&1
ESI_RANK_MODE=ballot timeout 300 $B > gpurun_out/g2_w2_ballot.json 2>&1
ESI_K2=block timeout 300 $B > gpurun_out/g2_block.json 2>&1
ESI_K2=block ESI_RANK_MODE=ballot timeout 300 $B > gpurun_out/g2_block_ballot.json 2>&1
for f in gpurun_out/g2_*.json; do echo $f; python -c "
import json,sys
for l in open('$f'):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(' ', d.get('value'), d.get('ms_per_step'), d.get('step_roofline',{}).get('kernel_ms_per_step'))
"; done
