# grid rule for AoS: BOYS_GRID_TILES 1 / 2, f64 and f32
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 1 2; do
  LAYOUT=aos BOYS_GRID_TILES=$v timeout 600 python tools/grid_rule.py "0,2,4,8,12,16:20,24" >> $out 2>&1
  LAYOUT=aos DTYPE=f32 BOYS_GRID_TILES=$v timeout 600 python tools/grid_rule.py "0,4,8,16:24" >> $out 2>&1
done; done
cat $out
