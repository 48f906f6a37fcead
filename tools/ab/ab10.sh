mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
BOYS_SOA_PPT=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dense_all_orders or sizes or config_inputs or host_path or domain" > gpurun_out/pytest_ppt2.log 2>&1
echo "PPT=2 pytest rc=$?" >> $out; tail -n 1 gpurun_out/pytest_ppt2.log >> $out
grep -q "rc=[1-9]" $out && { cat $out; exit 1; }
extras() {
  env "$@" timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | grep '^{' | \
    python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); c=d["configs"]["cfg1"]; print("cfg1", sys.argv[1:], c["roofline"]["frac"], c["roofline"]["launch_ms"])' "$@" >> $out
}
for rep in 1 2; do extras BOYS_SOA_PPT=1; extras BOYS_SOA_PPT=2; done
cat $out
