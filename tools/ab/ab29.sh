# grid rule sweep over SoA orders: BOYS_GRID_TILES 1 (one block per tile) / 2 (persistent)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 1 2; do BOYS_GRID_TILES=$v timeout 600 python tools/grid_rule.py "0,1,2,3,4,6,8,10,12,14,16:20,22,24" >> $out 2>&1; done; done
cat $out
