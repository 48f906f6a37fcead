# cfg5 (n=12 AoS): pair kernel single-buffered at 4 blocks/SM (libboys_p1.so + BOYS_AOS_PAIR=1) vs default
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f clk=%s" % (r["frac"], r["launch_ms"], d["clocks"]["sm_mhz"]))')" >> $out
}
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do
  run cfg5 BOYS_LIB=$L/libboys.so
  run cfg5 BOYS_LIB=$L/libboys_p1.so BOYS_AOS_PAIR=1
  echo "p1 $(BOYS_LIB=$L/libboys_p1.so BOYS_AOS_PAIR=1 LAYOUT=aos timeout 300 python tools/grid_rule.py "9,10,11,12:24" | tail -1)" >> $out
  echo "def $(BOYS_LIB=$L/libboys.so LAYOUT=aos timeout 300 python tools/grid_rule.py "9,10,11,12:24" | tail -1)" >> $out
done
cat $out
