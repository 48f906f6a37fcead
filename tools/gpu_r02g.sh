mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -q -m gpu -x -k "split" > gpurun_out/pytest_split.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_split.log; tail -n 2 gpurun_out/pytest_split.log
timeout 300 python tools/split_rate.py > gpurun_out/split_rate.jsonl 2>&1; cat gpurun_out/split_rate.jsonl
