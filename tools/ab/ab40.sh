# one comparison for both exp_neg_clamped selects + carried chunk element count (libboys.so) vs HEAD (libboys_prev.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
bash tools/ab/ab22.sh
L=$PWD/paper_2504_07637_b200
for rep in 1 2; do for lib in libboys.so libboys_prev.so; do
  echo "$lib $(BOYS_LIB=$L/$lib timeout 300 python tools/cfg1_stream.py 2>&1 | tail -1)" >> gpurun_out/ab.txt
done; done
tail -4 gpurun_out/ab.txt
