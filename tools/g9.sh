mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/g9_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/g9_pytest.log
