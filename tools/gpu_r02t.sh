mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -q -m gpu -x > gpurun_out/pytest_t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_t.log; tail -n 2 gpurun_out/pytest_t.log
for i in 1 2; do
BOYS_LIB=$PWD/ab_libs/libboys_old.so timeout 200 python tools/cfg1_stream.py
timeout 200 python tools/cfg1_stream.py
done
BOYS_LIB=$PWD/ab_libs/libboys_old.so timeout 800 python tools/order_sweep.py --out gpurun_out/sweep_old1.md > /dev/null 2>&1
timeout 800 python tools/order_sweep.py --out gpurun_out/sweep_new1.md > /dev/null 2>&1
