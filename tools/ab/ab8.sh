mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 200 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
L=paper_2504_07637_b200
for rep in 1 2; do
  run cfg2 BOYS_LIB=$L/libboys.so; run cfg2 BOYS_LIB=$L/libboys_soa5.so; run cfg2 BOYS_LIB=$L/libboys_soa6.so
done
run cfg4 X=1; run cfg3 X=1
cat $out
