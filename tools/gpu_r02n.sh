mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -q -m gpu -x > gpurun_out/pytest_n.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_n.log; tail -n 2 gpurun_out/pytest_n.log
timeout 800 python tools/order_sweep.py --out gpurun_out/sweep_new.md > /dev/null 2>&1
BOYS_LIB=$PWD/ab_libs/libboys_old.so timeout 800 python tools/order_sweep.py --out gpurun_out/sweep_old.md > /dev/null 2>&1
echo done
