set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-kernel-timing"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_integrate_w2 -s 30 -c 1 -o gpurun_out/prof_w2 -f $CMD > gpurun_out/ncu_w2.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_partition -s 30 -c 1 -o gpurun_out/prof_k1 -f $CMD > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/g3_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
