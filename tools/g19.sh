mkdir -p gpurun_out/r02
O=gpurun_out/r02
B="python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation"
for RM in atomic peers ballot; do
  ESI_RANK_MODE=$RM timeout 300 $B --validation fused > $O/rank_$RM.json 2> $O/rank_$RM.err; echo "$RM rc=$?"
done
timeout 600 python bench.py --config c4t --steps 5 --warmup 3 > $O/bench_c4t.json 2> $O/bench_c4t.err; echo "c4t rc=$?"; tail -2 $O/bench_c4t.err
for f in $O/rank_*.json $O/bench_c4t.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['value']/1e9,2), 'G ev/s', round(d['ms_per_step'],3),'ms', d.get('step_roofline',{}).get('kernel_ms_per_step'), d.get('stages'))
PY
done
