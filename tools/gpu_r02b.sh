# Round 2, pass 2: GPU tests + ncu --set full of the kernels below roofline (ragged f64/f32, n=0).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/pytest_gpu.log
python tools/prof_kernels.py --configs cfg4,cfg4f32,cfg1 --launches 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ragged_kernel|dense" -c 3 \
    -o gpurun_out/prof_r02b python tools/prof_kernels.py --configs cfg4,cfg4f32,cfg1 --launches 1 > gpurun_out/ncu_r02b.log 2>&1
echo "ncu rc=$?"
