#!/bin/bash
# A/B of libesi variants on the single-GPU configs:  LIBS="ref cur" CFGS="c2 c3" bash tools/abc.sh
mkdir -p gpurun_out
for L in ${LIBS:-ref cur}; do
  if [ "$L" = cur ]; then P=paper_2508_02238_b200/libesi.so; else P=paper_2508_02238_b200/variants/libesi_$L.so; fi
  ESI_LIB_PATH=$P timeout 900 python tools/bench_configs.py ${CFGS:-c2 c3} > gpurun_out/abc_$L.jsonl 2> gpurun_out/abc_$L.err
  python -c "
import json
for l in open('gpurun_out/abc_$L.jsonl'):
    d=json.loads(l); print('%-8s %-10s %4s fps  %.3f ms  %.3g ev/s' % ('$L', d['config'], d['fps'], d['ms'], d['events_per_s']))" || tail -3 gpurun_out/abc_$L.err
done
