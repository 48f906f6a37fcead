mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/pytest_gpu.log
timeout 200 python tools/cfg1_stream.py > gpurun_out/cfg1.jsonl 2>&1; cat gpurun_out/cfg1.jsonl
timeout 200 python tools/ragged_rate.py > gpurun_out/ragged_rate.jsonl 2>&1; cat gpurun_out/ragged_rate.jsonl
timeout 300 python tools/split_rate.py > gpurun_out/split_rate.jsonl 2>&1; cat gpurun_out/split_rate.jsonl
