mkdir -p gpurun_out
timeout 120 python tools/prof_kernels.py --configs cfg4,cfg4f32 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ragged_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_ragged_cur -f python tools/prof_kernels.py --configs cfg4 --launches 2 > gpurun_out/ncu_rg.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ragged_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_ragged_f32 -f python tools/prof_kernels.py --configs cfg4f32 --launches 2 > gpurun_out/ncu_rg32.log 2>&1
echo rc=$?
