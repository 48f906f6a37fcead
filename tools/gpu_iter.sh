# build-free iteration on the GPU box: tests, smoke, bench variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for nb in 1 2; do
  BOYS_AOS_NBUF=$nb timeout 600 python bench.py --steps 200 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_nbuf$nb.log 2>&1
  echo "bench nbuf=$nb rc=$?" >> gpurun_out/bench_nbuf$nb.log
done
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
