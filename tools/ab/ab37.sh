# fast-path rcp/sqrt self-test, ragged parity, then A/B: libboys.so (branch-free CR fast paths
# in the ragged chunks) vs libboys_prev.so
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ieee.py -q -x > gpurun_out/pytest_ieee.log 2>&1; echo "ieee rc=$?" >> gpurun_out/pytest_ieee.log
tail -3 gpurun_out/pytest_ieee.log
timeout 600 python -m pytest tests -q -x -m gpu -k "ragged or smoke or graph" > gpurun_out/pytest_ragged.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ragged.log
tail -2 gpurun_out/pytest_ragged.log
bash tools/ab/ab22.sh
