# paired SoA kernel, orders >= 11: 4 resident blocks (64 regs, some spill) vs 3 (80 regs) (libboys_h3.so)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for lib in libboys.so libboys_h3.so; do
  echo "$lib $(BOYS_LIB=$L/$lib timeout 300 python tools/grid_rule.py "11,12,13,14,15,16,20,24,36:22,24" 2>&1 | tail -1)" >> $out
done; done
cat $out
