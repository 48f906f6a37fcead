mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hermite.py tests/test_gpu_boundary.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_h.log; tail -n 2 gpurun_out/pytest_h.log
timeout 600 python bench.py --steps 5 --warmup 3 --extras hermite,cfg2 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/bench_h.jsonl 2> gpurun_out/bench_h.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_h.jsonl').read().strip().splitlines()[-1])
print({k:(v.get('value'),v.get('ms_per_step'),v.get('roofline',{}).get('frac'),v.get('l2'),v.get('accuracy')) for k,v in d['configs'].items()})"
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"hermite" -s 1 -c 1 -o gpurun_out/prof_hermite python -c "
import torch
from paper_2504_07637_b200 import hermite_coulomb, workloads as W
b=W.shell_pairs(4096, seed=21, device='cuda'); k=W.shell_pairs(4096, seed=22, device='cuda')
for _ in range(2): hermite_coulomb(4, b, k, check=False)
torch.cuda.synchronize()" > gpurun_out/ncu_h.log 2>&1; echo "ncu rc=$?"
