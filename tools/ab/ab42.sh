# split kernel with the AoS staging + bulk store (libboys.so) vs direct strided stores (libboys_prev.so)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "split or smoke" 2>&1 | tail -1
L=$PWD/paper_2504_07637_b200
for lib in libboys.so libboys_prev.so; do
  BOYS_LIB=$L/$lib timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | grep '^{' | \
    python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); s=d["configs"]["split"]; print("'$lib'", s.get("ms_per_step"), s.get("roofline",{}).get("frac"), s.get("error"))'
done
