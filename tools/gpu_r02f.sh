mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ieee.py tests/test_gpu_properties.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/pytest_dense.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_dense.log; tail -n 2 gpurun_out/pytest_dense.log
for i in 1 2; do timeout 200 python tools/cfg1_stream.py >> gpurun_out/cfg1.jsonl 2>&1; done
timeout 200 python tools/n0_probe.py >> gpurun_out/cfg1.jsonl 2>&1
cat gpurun_out/cfg1.jsonl
