# A/B in the cfg1 graph-stream measurement: persistent grid (default) vs one block per tile
# (BOYS_GRID_TILES=1) vs 6 resident blocks for n <= 1 (BOYS_SOA0_MINB=6)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do
  for v in "BOYS_PDL=1" "BOYS_GRID_TILES=1" "BOYS_SOA0_MINB=6"; do
    echo "$v $(env $v timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> $out
  done
done
cat $out
