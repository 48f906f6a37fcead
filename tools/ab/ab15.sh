mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for wt in 128 512; do
  BOYS_RAGGED_WIN=1 BOYS_RAGGED_WT=$wt timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "ragged" > gpurun_out/pytest_wt$wt.log 2>&1
  echo "WT=$wt pytest rc=$?" >> $out; tail -n 1 gpurun_out/pytest_wt$wt.log >> $out
done
grep -q "rc=[1-9]" $out && { cat $out; exit 1; }
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))')" >> $out
}
for wt in 128 256 512; do run cfg4 BOYS_RAGGED_WIN=1 BOYS_RAGGED_WT=$wt; run cfg4f32 BOYS_RAGGED_WIN=1 BOYS_RAGGED_WT=$wt; done
run cfg4 BOYS_RAGGED_WIN=0
cat $out
