mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 50 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/torchrun1.jsonl 2> gpurun_out/torchrun1.err
echo "torchrun ours rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/torchrun1_ref.jsonl 2> gpurun_out/torchrun1_ref.err
echo "torchrun ref rc=$?"
tail -c 1500 gpurun_out/torchrun1.jsonl; tail -c 600 gpurun_out/torchrun1_ref.jsonl; tail -5 gpurun_out/torchrun1.err
