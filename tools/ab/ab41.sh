# ragged code footprint: slow path as one copy (libboys.so) and + out-of-line drain (libboys_b.so)
# vs HEAD (libboys_prev.so)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "ragged or smoke" 2>&1 | tail -1
BOYS_LIB=$PWD/paper_2504_07637_b200/libboys_b.so timeout 600 python -m pytest tests -q -x -m gpu -k "ragged" 2>&1 | tail -1
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))')" >> $out
}
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for lib in libboys.so libboys_b.so libboys_prev.so; do
  run cfg4 BOYS_LIB=$L/$lib
  run cfg4f32 BOYS_LIB=$L/$lib
done; done
cat $out
