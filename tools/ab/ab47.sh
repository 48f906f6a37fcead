# AoS with two points per thread (BOYS_AOS_PAIR=1; orders whose double-buffered 512-point tile fits) vs default
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_knobs.py -q -x -k "AOS_PAIR or defaults" 2>&1 | tail -1 >> $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f clk=%s" % (r["frac"], r["launch_ms"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do for v in 0 1; do
  run cfg5 BOYS_AOS_PAIR=$v
  echo "AOS_PAIR=$v $(LAYOUT=aos BOYS_AOS_PAIR=$v timeout 300 python tools/grid_rule.py "2,4,6,8,10,12:24" 2>&1 | tail -1)" >> $out
done; done
cat $out
