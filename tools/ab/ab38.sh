# paired SoA kernel: shared fast-path checks for div/sqrt/rcp (libboys.so) vs per-op intrinsics
# (libboys_prev.so); plus the fast-path bit-identity test (rcp/sqrt/div)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ieee.py -q -x 2>&1 | tail -2
timeout 600 python -m pytest tests -q -x -m gpu -k "dense or soa or smoke or graph or host" 2>&1 | tail -2
out=gpurun_out/ab.txt; : > $out
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for lib in libboys.so libboys_prev.so; do
  echo "$lib $(BOYS_LIB=$L/$lib timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> $out
  BOYS_LIB=$L/$lib timeout 300 python tools/grid_rule.py "0,2,4,8,12,16:24" >> $out 2>&1
done; done
cat $out
