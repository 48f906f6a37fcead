# AoS register rows for n = 2..6 (BOYS_AOS_VEC=1; P = 2 libboys.so, P = 4 libboys_v4.so) vs defaults
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
BOYS_AOS_VEC=1 timeout 600 python tests/knob_parity.py 2>&1 | tail -1 >> $out
BOYS_LIB=$PWD/paper_2504_07637_b200/libboys_v4.so BOYS_AOS_VEC=1 timeout 600 python tests/knob_parity.py 2>&1 | tail -1 >> $out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for v in "libboys.so -1" "libboys.so 1" "libboys_v4.so 1"; do
  set -- $v
  echo "$1 VEC=$2 $(BOYS_LIB=$L/$1 BOYS_AOS_VEC=$2 LAYOUT=aos timeout 300 python tools/grid_rule.py "2,3,4,5,6:24" | tail -1)" >> $out
  echo "$1 VEC=$2 $(BOYS_LIB=$L/$1 BOYS_AOS_VEC=$2 LAYOUT=aos DTYPE=f32 timeout 300 python tools/grid_rule.py "2,3,4,5,6:24" | tail -1)" >> $out
done; done
cat $out
