# ragged: f64 4 / f32 5 elements per lane with 9 or 8 staged values per element (smem for 2 blocks/SM)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))')" >> $out
}
L=$PWD/paper_2504_07637_b200
for lib in libboys_r49.so libboys_r48.so; do
  BOYS_LIB=$L/$lib timeout 300 python -m pytest tests -q -x -m gpu -k "ragged_bit_exact or ragged_cfg4 or staging or ragged_random" 2>&1 | tail -1 >> $out
done
for rep in 1 2; do for lib in libboys.so libboys_r49.so libboys_r48.so; do
  run cfg4 BOYS_LIB=$L/$lib
  run cfg4f32 BOYS_LIB=$L/$lib
done; done
cat $out
