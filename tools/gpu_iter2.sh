mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 200 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
run cfg3 X=1; run cfg5 X=1; run cfg2 BOYS_SOA_TMA=0; run cfg2 BOYS_SOA_TMA=1; run cfg4 X=1; run cfg4f32 X=1; run cfg1 X=1
cat $out
BOYS_TABLE1_POINTS=1048576 BOYS_TABLE1_REPORT=gpurun_out/table1_2p20.json timeout 2400 \
  python -m pytest tests/test_table1_scan.py -x -q -m gpu > gpurun_out/table1.log 2>&1
echo "table1 rc=$?" >> gpurun_out/table1.log; tail -n 3 gpurun_out/table1.log
