# paired SoA kernel n <= 1: resident-block target (libboys_mK.so built with -DBOYS_PAIR_MINB_SMALL=K)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for lib in libboys_m5.so libboys_m4.so libboys_m3.so; do
  echo "$lib $(BOYS_LIB=$L/$lib timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> $out
  BOYS_LIB=$L/$lib timeout 300 python tools/grid_rule.py "0,1:22,24" >> $out 2>&1
done; done
cat $out
