# host-buffer pipeline chunk size (BOYS_HOST_CHUNK_LOG2 20 / 22 / 23 / 24): cfg3 e2e
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for c in 22 20 23 24; do
  echo "chunk=2^$c $(BOYS_HOST_CHUNK_LOG2=$c timeout 300 python bench.py --steps 3 --warmup 3 --no-extras --e2e-steps 3 --cpu-seconds 0 2>/dev/null | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"])')" >> $out
done; done
cat $out
