mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
extras() {   # per-config extras line (cfg1 is timed with the 1 GiB flush, kernel only)
  env "$@" timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | grep '^{' | \
    python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); c=d["configs"]["cfg1"]; print("cfg1", sys.argv[1:], c["roofline"]["frac"], c["roofline"]["launch_ms"])' "$@" >> $out
}
for rep in 1 2; do extras BOYS_GRID_TILES=0; extras BOYS_GRID_TILES=1; extras BOYS_GRID_TILES=0 BOYS_SOA0_MINB=6; done
cat $out
