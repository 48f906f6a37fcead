# same-box A/B of kernel variants (env knobs read by libboys at first launch)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
run() {  # env... -- config
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 200 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do
for f in 0 1 2 3; do for nb in 1 2; do run cfg3 BOYS_DENSE_FLAGS=$f BOYS_AOS_NBUF=$nb; done; done
for f in 0 1; do run cfg2 BOYS_DENSE_FLAGS=$f; run cfg1 BOYS_DENSE_FLAGS=$f; done
for v in 1 2; do run cfg4 BOYS_RAGGED_V=$v; run cfg4f32 BOYS_RAGGED_V=$v; done
done
cat $out
python tools/prof_kernels.py --configs cfg4 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
BOYS_RAGGED_V=2 ncu --set full --clock-control none --import-source on -k regex:"ragged_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_ragged_v2 python tools/prof_kernels.py --configs cfg4 --launches 2 > gpurun_out/ncu_ragged.log 2>&1
