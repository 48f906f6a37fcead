# cfg1 two ways (graph-replayed stream of 32 batches; L2-flushed single launch) + the full extras line
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 3 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/bench_extras.jsonl 2> gpurun_out/bench_extras.err
echo "rc=$?" >> gpurun_out/bench_extras.err; tail -3 gpurun_out/bench_extras.err
