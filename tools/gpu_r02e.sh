mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -q -m gpu -x -k "ragged" > gpurun_out/pytest_ragged.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_ragged.log; tail -n 3 gpurun_out/pytest_ragged.log
timeout 120 python tools/ragged_rate.py > gpurun_out/ragged_rate.jsonl 2>&1
cat gpurun_out/ragged_rate.jsonl
