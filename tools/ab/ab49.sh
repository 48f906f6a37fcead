# SoA n <= 1 with four adjacent points per thread (BOYS_SOA_QUAD=1; MINB 3 / 2 / 4 builds) vs the pair kernel
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 600 python -m pytest tests/test_gpu_knobs.py -q -x -k "QUAD" 2>&1 | tail -1 >> $out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do
  for v in "libboys.so 0" "libboys.so 1" "libboys_q2.so 1" "libboys_q4.so 1"; do
    set -- $v
    echo "$1 QUAD=$2 $(BOYS_LIB=$L/$1 BOYS_SOA_QUAD=$2 timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> $out
    echo "$1 QUAD=$2 $(BOYS_LIB=$L/$1 BOYS_SOA_QUAD=$2 timeout 300 python tools/grid_rule.py "0,1:22,24" 2>&1 | tail -1)" >> $out
  done
done
cat $out
