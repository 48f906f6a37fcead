mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 300 python bench.py --config $cfg --steps 200 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do
  for v in "BOYS_AOS_MINB=4" "BOYS_AOS_MINB=6" "BOYS_AOS_NBUF=2"; do run cfg3 $v; run cfg5 $v; done
  run cfg2 X=1; run cfg1 X=1; run cfg4 X=1; run cfg4f32 X=1
done
cat $out
python tools/prof_kernels.py --configs cfg4,cfg3 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
BOYS_AOS_MINB=6 ncu --set full --clock-control none --import-source on -k regex:"ragged_kernel|dense_kernel" -s 1 -c 3 \
    -o gpurun_out/prof_v3 python tools/prof_kernels.py --configs cfg4,cfg3 --launches 2 > gpurun_out/ncu_v3.log 2>&1
