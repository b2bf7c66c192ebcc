mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_slice_maps.py -m gpu -q -x > gpurun_out/g16_slice.log 2>&1; echo "slice rc=$?"
tail -30 gpurun_out/g16_slice.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g16_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g16_pytest.log
