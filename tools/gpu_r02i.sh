mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x --durations=10 > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log; grep -E "passed|failed|rc=|s call" gpurun_out/pytest_full.log | head -20
