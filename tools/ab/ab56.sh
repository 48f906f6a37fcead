# AoS n = 1, 3 with register rows and direct 16-byte stores (BOYS_AOS_VEC=1; P = 4 libboys.so, P = 2 libboys_v2.so)
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 600 python -m pytest tests/test_gpu_knobs.py -q -x -k "AOS_VEC" 2>&1 | tail -1 >> $out
BOYS_LIB=$PWD/paper_2504_07637_b200/libboys_v2.so BOYS_AOS_VEC=1 timeout 600 python tests/knob_parity.py 2>&1 | tail -1 >> $out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for v in "libboys.so 0" "libboys.so 1" "libboys_v2.so 1"; do
  set -- $v
  echo "$1 VEC=$2 $(BOYS_LIB=$L/$1 BOYS_AOS_VEC=$2 LAYOUT=aos timeout 300 python tools/grid_rule.py "1,3:22,24" | tail -1)" >> $out
  echo "$1 VEC=$2 $(BOYS_LIB=$L/$1 BOYS_AOS_VEC=$2 LAYOUT=aos DTYPE=f32 timeout 300 python tools/grid_rule.py "1,3:24" | tail -1)" >> $out
done; done
cat $out
