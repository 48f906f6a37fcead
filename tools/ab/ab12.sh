mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 200 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
L=paper_2504_07637_b200
for rep in 1 2; do for c in cfg2 cfg3 cfg5; do run $c BOYS_LIB=$L/libboys_prev.so; run $c BOYS_LIB=$L/libboys.so; done; done
cat $out
