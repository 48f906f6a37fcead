# A/B: paired SoA kernel (two adjacent points per thread, 16-byte loads/stores) BOYS_SOA_PAIR=1 vs 0
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 1 0; do
  echo "PAIR=$v $(BOYS_SOA_PAIR=$v timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> $out
  BOYS_SOA_PAIR=$v timeout 600 python tools/grid_rule.py "0,1,2,4,6,8,10,12,14,16:22,24" >> $out 2>&1
  BOYS_SOA_PAIR=$v DTYPE=f32 timeout 600 python tools/grid_rule.py "0,2,4,8,12,16:24" >> $out 2>&1
done; done
cat $out
