# grid rule sweep: f32 SoA orders, and f64 n=5/11 at 2^24: BOYS_GRID_TILES 1 / 2
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 1 2; do
  DTYPE=f32 BOYS_GRID_TILES=$v timeout 600 python tools/grid_rule.py "0,2,4,6,8,10,12,16:22,24" >> $out 2>&1
  BOYS_GRID_TILES=$v timeout 600 python tools/grid_rule.py "5,7,9,11,13:24" >> $out 2>&1
done; done
cat $out
