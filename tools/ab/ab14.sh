mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
for v in 0 1; do BOYS_RAGGED_WIN=$v timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -m gpu -k "ragged" 2>&1 | tail -n 1; done
timeout 300 python bench.py --steps 100 --warmup 5 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/bench_extras.jsonl 2>&1
python3 -c "
import json
d=json.loads(open('gpurun_out/bench_extras.jsonl').read().strip().split(chr(10))[-1])
print('cfg3', d['roofline']['frac'], d['roofline']['launch_ms'])
for k,v in d['configs'].items(): print(k, v['roofline']['frac'], v['roofline']['launch_ms'])
"
