mkdir -p gpurun_out/r02
timeout 900 ncu --set full --clock-control none --import-source on -k regex:esi_slice_summary -s 5 -c 1 -o gpurun_out/r02/ncu_slice -f python tools/bench_slices.py > gpurun_out/r02/ncu_slice.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r02/ncu_slice.log
