#!/bin/bash
# streaming-latency A/B:  LIBS="ref cur" bash tools/lat.sh
for L in ${LIBS:-ref cur}; do
  if [ "$L" = cur ]; then P=paper_2508_02238_b200/libesi.so; else P=paper_2508_02238_b200/variants/libesi_$L.so; fi
  ESI_LIB_PATH=$P timeout 600 python -c "
import sys, json; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, argparse
r = bench.run_latency(argparse.Namespace())
print('$L', json.dumps({k:(round(v['mean_ms_per_frame'],3), round(v['p99_ms_per_frame'],3), round(v['render_p99_ms'],3)) for k,v in r.items()}))
" 2>&1 | tail -1
done
