# AoS: generic multi-point kernel with P=2 (defaults) and P=4 (BOYS_AOS_QUAD=1) vs the earlier pair numbers
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_knobs.py -q -x -k "AOS or defaults" 2>&1 | tail -1 >> $out
timeout 900 python -m pytest tests -q -x -m gpu -k "dense or aos or sizes" 2>&1 | tail -1 >> $out
for rep in 1 2; do for v in 0 1; do
  echo "AOS_QUAD=$v $(LAYOUT=aos BOYS_AOS_QUAD=$v timeout 300 python tools/grid_rule.py "1,2,3,8:22,24" 2>&1 | tail -1)" >> $out
  echo "AOS_QUAD=$v $(LAYOUT=aos DTYPE=f32 BOYS_AOS_QUAD=$v timeout 300 python tools/grid_rule.py "1,2,4,8,16:24" 2>&1 | tail -1)" >> $out
done; done
cat $out
