# same-box A/B: current libboys.so vs libboys_prev.so (BOYS_LIB override)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))')" >> $out
}
for rep in 1 2; do
  run cfg4 BOYS_LIB=$PWD/paper_2504_07637_b200/libboys.so
  run cfg4 BOYS_LIB=$PWD/paper_2504_07637_b200/libboys_prev.so
  run cfg4f32 BOYS_LIB=$PWD/paper_2504_07637_b200/libboys.so
  run cfg4f32 BOYS_LIB=$PWD/paper_2504_07637_b200/libboys_prev.so
done
cat $out
