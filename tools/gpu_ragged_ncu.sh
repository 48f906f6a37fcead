# Ragged kernels: ncu --set full with source, key issue/stall metrics, per-source-line attribution.
# usage: gpu_ragged_ncu.sh [configs...]   (default cfg4 cfg4f32)
mkdir -p gpurun_out
CFGS=${@:-cfg4 cfg4f32}
cd /tmp && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2504_07637_b200/libboys.so > /dev/null 2>&1
cd $GRAFT_REPO_ROOT
nvdisasm --print-line-info /tmp/ragged.sm_100a.cubin > /tmp/ragged.txt 2>/dev/null
nvdisasm -gi /tmp/ragged.sm_100a.cubin > /tmp/ragged_gi.txt 2>/dev/null
for cfg in $CFGS; do
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:"ragged_kernel" -s 1 -c 1 \
    -o /tmp/prof_$cfg python tools/prof_kernels.py --configs $cfg --launches 2 > gpurun_out/ncu_$cfg.log 2>&1
echo "ncu $cfg rc=$?"
ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv > /tmp/src_$cfg.csv 2>/dev/null
ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/raw_$cfg.csv 2>/dev/null
python tools/ncu_keys.py gpurun_out/raw_$cfg.csv | tee gpurun_out/keys_$cfg.txt
F=$(grep -o "^\.text\._ZN4boys13ragged_kernelI$([ $cfg = cfg4 ] && echo d || echo f)[A-Za-z0-9_]*" /tmp/ragged.txt | head -1 | sed 's/^\.text\.//')
python tools/sass_lines.py /tmp/src_$cfg.csv /tmp/ragged.txt $F ragged_kernel 60 > gpurun_out/lines_$cfg.txt 2>&1
# the same counts attributed to the outermost (call-site) line
python tools/sass_lines.py /tmp/src_$cfg.csv /tmp/ragged_gi.txt $F ragged_kernel 70 > gpurun_out/lines_outer_$cfg.txt 2>&1
done
