mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-kernel-timing --no-latency --no-alt-validation --validation fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_integrate_px -s 30 -c 1 -o gpurun_out/prof_px1 -f $CMD > gpurun_out/ncu_px1.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_px1.log
