# staged AoS with four points per thread (BOYS_AOS_QUAD4=1, register rows off) vs defaults, f64 n=2,3 and f32 n=2..8
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
timeout 600 python -m pytest tests/test_gpu_knobs.py -q -x -k "QUAD4" 2>&1 | tail -1 >> $out
for rep in 1 2; do for v in "-1 -1" "1 0"; do
  set -- $v
  echo "QUAD4=$1 $(BOYS_AOS_QUAD4=$1 BOYS_AOS_VEC=$2 LAYOUT=aos timeout 300 python tools/grid_rule.py "2,3:24" | tail -1)" >> $out
  echo "QUAD4=$1 $(BOYS_AOS_QUAD4=$1 BOYS_AOS_VEC=$2 LAYOUT=aos DTYPE=f32 timeout 300 python tools/grid_rule.py "2,3,4,5,6,8:24" | tail -1)" >> $out
done; done
cat $out
