#!/bin/bash
# streaming latency with and without the sync-free one-chunk render (ESI_SYNC_PLAN=1 reads the plan back)
for SP in 1 0 1 0; do
  ESI_SYNC_PLAN=$SP timeout 600 python -c "
import sys, json; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, argparse
r = bench.run_latency(argparse.Namespace())
print('sync_plan=$SP', json.dumps({k:(round(v['mean_ms_per_frame'],3), round(v['p99_ms_per_frame'],3), round(v['render_mean_ms'],3), round(v['render_p99_ms'],3)) for k,v in r.items()}))
" 2>&1 | tail -1
done
