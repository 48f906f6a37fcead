mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -k "ragged" > gpurun_out/pytest_s.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_s.log; tail -n 2 gpurun_out/pytest_s.log
for i in 1 2; do
BOYS_LIB=$PWD/ab_libs/libboys_old.so timeout 200 python tools/ragged_rate.py
timeout 200 python tools/ragged_rate.py
done
