# Round-2 evidence, part B: ncu --set full of every config's kernel (second launch each);
# the report is summarised on the box (raw-page CSV + traffic json) and only the
# headline cfg3 capture (with source) comes back, to stay under gpurun's 64 MiB.
mkdir -p gpurun_out
CF=cfg3,cfg2,cfg1,cfg4,cfg4f32,cfg5,split,hermite
timeout 300 python tools/prof_kernels.py --configs $CF --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu -f --set full --clock-control none \
    -k regex:"dense_kernel|dense_soa_pair|dense_soa_quad|ragged_kernel|split_kernel|hermite_kernel" -c 16 \
    -o /tmp/prof_r02 python tools/prof_kernels.py --configs $CF --launches 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu -i /tmp/prof_r02.ncu-rep --page raw --csv > gpurun_out/prof_r02_raw.csv 2>&1
python tools/summarize_ncu.py full /tmp/prof_r02.ncu-rep > gpurun_out/prof_r02_summary.md 2>&1
python tools/traffic_json.py /tmp/prof_r02.ncu-rep $CF "ncu --set full, round-2 kernels, second launch of each config (tools/gpu_r02_ncu.sh)" > gpurun_out/traffic.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"dense_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_r02_cfg3 python tools/prof_kernels.py --configs cfg3 --launches 2 > gpurun_out/ncu_cfg3.log 2>&1
echo "ncu cfg3 rc=$?"; ls -la gpurun_out
