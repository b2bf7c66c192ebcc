#!/bin/bash
# A/B of K2 variants: ESI_AB="libesi_base.so libesi_a.so ..." (built in-tree), configs c3 c4 c4@1000, two passes
mkdir -p gpurun_out
for pass in 1 2; do
  for L in ${ESI_AB}; do
    echo "== $L"; ESI_LIB_PATH=$PWD/paper_2508_02238_b200/$L timeout 600 python tools/bench_configs.py ${AB_CONFIGS:-c3 c4 c4@1000} 2>&1 | tail -3 | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print('  %s@%d %.3f ms %.2f Gev/s' % (d['config'], d['fps'], d['ms'], d['events_per_s'] / 1e9))
    except Exception: print(l.rstrip())"
  done
done
