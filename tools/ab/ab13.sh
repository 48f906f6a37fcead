mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for v in 1 0; do
  BOYS_RAGGED_WIN=$v timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_accuracy.py -x -q -m gpu -k "ragged" > gpurun_out/pytest_win$v.log 2>&1
  echo "WIN=$v pytest rc=$?" >> $out; tail -n 1 gpurun_out/pytest_win$v.log >> $out
done
grep -q "rc=[1-9]" $out && { cat $out; grep -E "Error|assert" gpurun_out/pytest_win1.log | head -5; exit 1; }
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do for v in 0 1; do run cfg4 BOYS_RAGGED_WIN=$v; run cfg4f32 BOYS_RAGGED_WIN=$v; done; done
cat $out
