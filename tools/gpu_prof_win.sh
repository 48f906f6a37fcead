mkdir -p gpurun_out
BOYS_RAGGED_WIN=1 timeout 120 python tools/prof_kernels.py --configs cfg4 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
BOYS_RAGGED_WIN=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ragged_win" -s 1 -c 1 \
    -o gpurun_out/prof_win python tools/prof_kernels.py --configs cfg4 --launches 2 > gpurun_out/ncu_win.log 2>&1
echo rc=$?
