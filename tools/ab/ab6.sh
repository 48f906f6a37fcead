mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
out=gpurun_out/ab.txt; : > $out
run() {
  local cfg=$1; shift
  local line
  line=$(env "$@" timeout 120 python bench.py --config $cfg --steps 200 --warmup 5 --no-extras --e2e-steps 0 --cpu-seconds 0 2>&1 | grep '^{')
  echo "$cfg $* :: $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("frac=%.4f launch_ms=%.4f val=%.4g clk=%s" % (r["frac"], r["launch_ms"], d["value"], d["clocks"]["sm_mhz"]))')" >> $out
}
for rep in 1 2; do run cfg1 BOYS_SOA0_MINB=8; run cfg1 BOYS_SOA0_MINB=6; done
timeout 300 python bench.py --steps 100 --warmup 5 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/bench_extras.jsonl 2>&1
python3 -c "
import json
d=json.loads(open('gpurun_out/bench_extras.jsonl').read().strip().split(chr(10))[-1])
for k,v in d['configs'].items(): print(k, v['roofline']['frac'], v['roofline']['launch_ms'])
" >> $out
cat $out
