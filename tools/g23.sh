mkdir -p gpurun_out/r02
timeout 600 python tools/bench_slices.py > gpurun_out/r02/slices.json 2> gpurun_out/r02/slices.err; echo "slices rc=$?"; tail -3 gpurun_out/r02/slices.err; cat gpurun_out/r02/slices.json
timeout 600 python -m pytest tests/test_slice_maps.py -m gpu -q > gpurun_out/r02/slice_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02/slice_tests.log
