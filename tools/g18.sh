# round-2 measurement set (N = 1): tests, bench lines, configs, variants, ncu
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi > $O/nvsmi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1; nproc >> $O/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -2 $O/bench.err
timeout 600 python bench.py --fps 1000 --steps 10 --e2e-steps 0 --no-cpu-baseline --no-latency > $O/bench_1000fps.json 2> $O/bench_1000fps.err; echo "b1000 rc=$?"
timeout 600 python bench.py --config c4t --steps 5 --warmup 3 > $O/bench_c4t.json 2> $O/bench_c4t.err; echo "c4t rc=$?"; tail -2 $O/bench_c4t.err
timeout 900 python bench.py --config c5a --steps 2 --warmup 3 > $O/bench_c5a.json 2> $O/bench_c5a.err; echo "c5a rc=$?"; tail -2 $O/bench_c5a.err
timeout 900 python bench.py --config c5b --steps 3 --warmup 3 > $O/bench_c5b.json 2> $O/bench_c5b.err; echo "c5b rc=$?"; tail -2 $O/bench_c5b.err
timeout 900 python tools/bench_configs.py c1 c2 c3 c4 c4@1000 c4:decay_kind=1 c4:decay_first=1 c4:decay_kind=2 c4:state_unclamped=1 > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"; tail -2 $O/configs.err
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-latency --no-alt-validation --no-kernel-timing"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_integrate_kernel -s 30 -c 1 -o $O/ncu_integrate -f $CMD > $O/ncu_integrate.log 2>&1; echo "ncu K2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_partition_kernel -s 30 -c 1 -o $O/ncu_partition -f $CMD > $O/ncu_partition.log 2>&1; echo "ncu K1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_validate -s 1 -c 1 -o $O/ncu_validate -f $CMD > $O/ncu_validate.log 2>&1; echo "ncu val rc=$?"
