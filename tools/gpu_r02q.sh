mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_q.log; tail -n 2 gpurun_out/pytest_q.log
timeout 800 python tools/order_sweep.py --out gpurun_out/r02_order_sweep.md > /dev/null 2>&1
timeout 200 python tools/cfg1_stream.py; timeout 300 python tools/dense_rate.py
