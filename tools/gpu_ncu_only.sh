mkdir -p gpurun_out
timeout 120 python tools/prof_kernels.py --configs cfg3,cfg2,cfg1,cfg4,cfg4f32,cfg5 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dense_kernel|ragged" -s 0 -c 12 \
    -o gpurun_out/prof_round python tools/prof_kernels.py --configs cfg3,cfg2,cfg1,cfg4,cfg4f32,cfg5 --launches 2 > gpurun_out/ncu_full.log 2>&1
echo rc=$?
