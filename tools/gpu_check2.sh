# full GPU suite with the current defaults, then ragged benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; rc=$?
tail -n 3 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && { grep -E "Error|assert|FAILED" gpurun_out/pytest_gpu.log | head -20; exit 1; }
for cfg in cfg4 cfg4f32; do
  timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{' | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["config"]["workload"], "frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))'
done
