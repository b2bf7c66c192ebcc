CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:esi_partition -s 10 -c 1 -o gpurun_out/prof_part $CMD > gpurun_out/ncu_part.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:esi_integrate -s 10 -c 1 -o gpurun_out/prof_int $CMD > gpurun_out/ncu_int.log 2>&1 ; \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:esi_ --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo done
