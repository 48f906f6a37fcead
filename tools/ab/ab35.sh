# ragged grid: resident blocks x BOYS_RAGGED_GRID_MULT (1 = persistent default)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f clk=%s" % (r["frac"], r["launch_ms"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do
  for m in 1 2 4 16 100000; do
    run cfg4 BOYS_RAGGED_GRID_MULT=$m
    run cfg4f32 BOYS_RAGGED_GRID_MULT=$m
  done
done
cat $out
