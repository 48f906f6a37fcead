# Round evidence: tests, smoke, default bench, reference arm, ncu launch list + full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_info.txt
timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
rc=$?; echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 > gpurun_out/bench_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-extras --e2e-steps 0 --cpu-seconds 0 > gpurun_out/ncu_launch.log 2>&1
timeout 120 python tools/prof_kernels.py --configs cfg3,cfg2,cfg1,cfg4,cfg4f32,cfg5 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dense_kernel|dense_soa_pair|dense_soa_quad|dense_aos_pair|ragged" -s 0 -c 12 \
    -o gpurun_out/prof_round python tools/prof_kernels.py --configs cfg3,cfg2,cfg1,cfg4,cfg4f32,cfg5 --launches 2 > gpurun_out/ncu_full.log 2>&1
echo done
