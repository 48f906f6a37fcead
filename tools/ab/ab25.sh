# same-box A/B: dense x prefetch (libboys.so: SoA on; libboys_pfaos.so: SoA+AoS on) vs libboys_prev.so (off)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 600 python -m pytest tests -q -x -m gpu -k "dense or soa or aos or smoke" > gpurun_out/pytest_dense.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dense.log
tail -2 gpurun_out/pytest_dense.log
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f clk=%s" % (r["frac"], r["launch_ms"], d["clocks"]["sm_mhz"]))')" >> $out
}
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do
  for cfg in cfg2 cfg3 cfg5; do
    for lib in libboys.so libboys_pfaos.so libboys_prev.so; do run $cfg BOYS_LIB=$L/$lib; done
  done
done
# cfg1 both ways via the full extras line
BOYS_LIB=$L/libboys.so timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/bench_extras.jsonl 2>&1
cat $out
