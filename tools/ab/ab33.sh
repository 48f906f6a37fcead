# paired SoA kernel grid: BOYS_PAIR_GRID 1 (per tile) vs 2 (persistent), orders 5..12, plus cfg2 via cfg1_stream
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 1 2; do
  echo "PAIR_GRID=$v $(BOYS_PAIR_GRID=$v timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> $out
  BOYS_PAIR_GRID=$v timeout 600 python tools/grid_rule.py "5,6,7,8,9,10,11,12:24" >> $out 2>&1
  BOYS_PAIR_GRID=$v DTYPE=f32 timeout 600 python tools/grid_rule.py "0,4,8,12,16:24" >> $out 2>&1
done; done
cat $out
