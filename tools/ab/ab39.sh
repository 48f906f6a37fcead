# ragged block size / register bound / staging: BOYS_RAGGED_CFG 0 (256 thr) / 1 (128) / 2 (128, <=96 regs) / 3 (128, <=96 regs, 8 staged values/elem)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))')" >> $out
}
for v in 0 1 2 3; do BOYS_RAGGED_CFG=$v timeout 300 python -m pytest tests -q -x -m gpu -k "ragged" 2>&1 | tail -1 >> $out; done
for rep in 1 2; do for v in 0 1 2 3; do
  run cfg4 BOYS_RAGGED_CFG=$v
  run cfg4f32 BOYS_RAGGED_CFG=$v
done; done
cat $out
