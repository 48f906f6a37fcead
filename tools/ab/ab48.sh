# AoS pair (BOYS_AOS_PAIR=1) vs default for f32 orders
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in 0 1; do
  echo "AOS_PAIR=$v $(LAYOUT=aos DTYPE=f32 BOYS_AOS_PAIR=$v timeout 300 python tools/grid_rule.py "1,2,4,8,12,16:24" 2>&1 | tail -1)" >> $out
done; done
cat $out
