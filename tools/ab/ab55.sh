# SoA split register bound: BOYS_SPLIT_SOA_MINB 1 (default, 134 regs) / 2 / 3 / 4
mkdir -p gpurun_out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for lib in libboys.so libboys_s2.so libboys_s3.so libboys_s4.so; do
  echo "$lib $(BOYS_LIB=$L/$lib timeout 300 python tools/split_rate.py | tail -1)"
done; done
