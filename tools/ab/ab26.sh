# A/B: programmatic dependent launch for dense kernels (BOYS_PDL=1 default vs 0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
out=gpurun_out/ab.txt; : > $out
for rep in 1 2 3; do
  for p in 1 0; do BOYS_PDL=$p timeout 300 python tools/cfg1_stream.py >> $out 2>&1; done
done
cat $out
