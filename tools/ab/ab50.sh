# four points per thread (BOYS_SOA_QUAD=1) vs the pair kernel for SoA n <= 5, f64 and f32
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 600 python -m pytest tests/test_gpu_knobs.py -q -x -k "QUAD" 2>&1 | tail -1 >> $out
for rep in 1 2; do for v in 0 1; do
  echo "QUAD=$v $(BOYS_SOA_QUAD=$v timeout 300 python tools/grid_rule.py "0,1,2,3,4,5:20,22,24" 2>&1 | tail -1)" >> $out
  echo "QUAD=$v $(DTYPE=f32 BOYS_SOA_QUAD=$v timeout 300 python tools/grid_rule.py "0,1,2,4,5:22,24" 2>&1 | tail -1)" >> $out
done; done
cat $out
