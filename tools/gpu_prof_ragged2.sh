# one ncu --set full capture of the ragged kernels (f64, f32) with source attribution
mkdir -p gpurun_out
python tools/prof_kernels.py --configs cfg4,cfg4f32 --launches 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ragged" -c 2 \
    -o gpurun_out/prof_ragged python tools/prof_kernels.py --configs cfg4,cfg4f32 --launches 1 > gpurun_out/ncu_ragged.log 2>&1
echo rc=$?
