# Per-line instruction / stall attribution of one kernel: ncu --set full with source.
# usage: gpu_lines.sh <config> <kernel regex> <cubin unit> <mangled-name substring>
mkdir -p gpurun_out
cfg=$1; kre=$2; unit=$3; sub=$4
cd /tmp && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2504_07637_b200/libboys.so > /dev/null 2>&1
cd $GRAFT_REPO_ROOT
nvdisasm --print-line-info /tmp/$unit.sm_100a.cubin > /tmp/$unit.txt 2>/dev/null
nvdisasm -gi /tmp/$unit.sm_100a.cubin > /tmp/${unit}_gi.txt 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:"$kre" -s 1 -c 1 \
    -o /tmp/prof_$cfg python tools/prof_kernels.py --configs $cfg --launches 2 > gpurun_out/ncu_$cfg.log 2>&1
echo "ncu $cfg rc=$?"
ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv > /tmp/src_$cfg.csv 2>/dev/null
ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/raw_$cfg.csv 2>/dev/null
cp /tmp/src_$cfg.csv gpurun_out/src_$cfg.csv; gzip -f gpurun_out/src_$cfg.csv; cp /tmp/${unit}_gi.txt gpurun_out/${unit}_gi.txt; gzip -f gpurun_out/${unit}_gi.txt
python tools/ncu_keys.py gpurun_out/raw_$cfg.csv | tee gpurun_out/keys_$cfg.txt
F=$(grep -o "^\.text\.[A-Za-z0-9_]*$sub[A-Za-z0-9_]*" /tmp/$unit.txt | head -1 | sed 's/^\.text\.//')
python tools/sass_lines.py /tmp/src_$cfg.csv /tmp/$unit.txt $F "$kre" 60 > gpurun_out/lines_$cfg.txt 2>&1
python tools/sass_lines.py /tmp/src_$cfg.csv /tmp/${unit}_gi.txt $F "$kre" 60 > gpurun_out/lines_outer_$cfg.txt 2>&1
# instruction mix actually executed
python - <<PY > gpurun_out/mix_$cfg.txt 2>&1
import csv, collections
rows=list(csv.reader(open('/tmp/src_$cfg.csv')))
hdr=None; agg=collections.Counter()
for r in rows:
    if 'Instructions Executed' in r and 'Source' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); op=d['Source'].split()
        if not op: continue
        o=op[1] if op[0].startswith('@') and len(op)>1 else op[0]
        try: agg[o.split('.')[0]]+=int(d['Instructions Executed'] or 0)
        except ValueError: pass
t=sum(agg.values()) or 1
print(t,'warp instructions')
for k,v in agg.most_common(30): print(f'{100*v/t:5.1f}%  {v:12d}  {k}')
PY
