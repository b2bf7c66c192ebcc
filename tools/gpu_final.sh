#!/bin/bash
# End-of-round GPU session: everything in gpu_all.sh plus the router and per-config benches.
bash tools/gpu_all.sh
for r in 1 2; do timeout 600 python tools/bench_route.py > gpurun_out/route_$r.json 2> gpurun_out/route_$r.err; echo "route$r rc=$?"; done
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
ESI_LIB_PATH=$PWD/paper_2508_02238_b200/libesi_checked.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_checked.log 2>&1; echo "checked rc=$?"
