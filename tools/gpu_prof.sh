set -x
mkdir -p gpurun_out
python tools/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dense_kernel|ragged_kernel" -s 0 -c 12 \
    -o gpurun_out/prof_r01 python tools/prof_kernels.py --launches 2 > gpurun_out/ncu_full.log 2>&1
python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
