mkdir -p gpurun_out
for i in 1 2; do
BOYS_LIB=$PWD/ab_libs/libboys_wide.so timeout 800 python tools/order_sweep.py --out gpurun_out/sweep_wide$i.md > /dev/null 2>&1
BOYS_LIB=$PWD/ab_libs/libboys_old.so timeout 800 python tools/order_sweep.py --out gpurun_out/sweep_old$i.md > /dev/null 2>&1
done
BOYS_LIB=$PWD/ab_libs/libboys_wide.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "all_orders or sizes" > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"
echo done
