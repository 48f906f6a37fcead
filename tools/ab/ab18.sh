# A/B: ragged warp-chunk kernel, elements per lane x register bound (MINB)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for v in "3 1" "4 3"; do
  set -- $v
  BOYS_RAGGED_WIN=0 BOYS_RAGGED_EPL=$1 BOYS_RAGGED_MINB=$2 timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -m gpu -k "ragged" > gpurun_out/pytest_epl$1_$2.log 2>&1
  echo "EPL=$1 MINB=$2 pytest rc=$?" >> $out; tail -n 1 gpurun_out/pytest_epl$1_$2.log >> $out
done
grep -q "rc=[1-9]" $out && { cat $out; exit 1; }
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f" % (r["frac"], r["launch_ms"]))')" >> $out
}
for mb in 1 3; do
  for epl in 1 2 3 4; do run cfg4 BOYS_RAGGED_WIN=0 BOYS_RAGGED_EPL=$epl BOYS_RAGGED_MINB=$mb; done
  for epl in 2 3 4 6 8; do run cfg4f32 BOYS_RAGGED_WIN=0 BOYS_RAGGED_EPL=$epl BOYS_RAGGED_MINB=$mb; done
done
cat $out
