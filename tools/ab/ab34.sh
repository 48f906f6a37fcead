# AoS knobs on cfg5 (n=12) and cfg3 (n=16): default (NBUF=2, MINB=4) vs NBUF=1 vs MINB=6
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f clk=%s" % (r["frac"], r["launch_ms"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do
  for cfg in cfg5 cfg3; do
    run $cfg BOYS_AOS_NBUF=2
    run $cfg BOYS_AOS_NBUF=1
    run $cfg BOYS_AOS_NBUF=1 BOYS_AOS_MINB=6
  done
done
cat $out
