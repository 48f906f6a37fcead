# grid rule: BOYS_GRID_TILES 0 (auto) / 1 (one block per tile) / 2 (persistent)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 0 1 2; do BOYS_GRID_TILES=$v timeout 300 python tools/grid_rule.py >> $out 2>&1; done; done
cat $out
