mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
BOYS_TABLE1_POINTS=1048576 BOYS_TABLE1_REPORT=gpurun_out/table1_2p20.json timeout 1800 \
  python -m pytest tests/test_table1_scan.py -x -q -m gpu > gpurun_out/table1.log 2>&1
echo "table1 rc=$?" >> gpurun_out/table1.log; tail -n 3 gpurun_out/table1.log
