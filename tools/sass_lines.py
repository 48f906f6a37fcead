"""Attribute ncu per-instruction counts (SASS page CSV) to source lines via
nvdisasm --print-line-info of the same cubin."""
import csv
import re
import sys
from collections import defaultdict

sass_csv, lines_txt, func, kname = sys.argv[1:5]
lines = open(lines_txt).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{func}:"))
insts, cur = [], (None, None)
for l in lines[start + 1:]:
    if l.startswith(".text.") or (l.startswith("\t.section") and insts):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        insts.append((cur, m.group(2)))
rows = list(csv.reader(open(sass_csv)))
blocks, b = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        b = [r[1]]
        blocks.append(b)
        continue
    if b is not None:
        b.append(r)
blk = next(b for b in blocks if kname in b[0])
hdr = blk[1]
data = [r for r in blk[2:] if len(r) == len(hdr)]
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
agg = defaultdict(lambda: [0, 0])
for k, r in enumerate(data[: len(insts)]):
    agg[insts[k][0]][0] += int(r[ii] or 0)
    agg[insts[k][0]][1] += int(r[si] or 0)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
src = {}
for fn in ("dense.cu", "ragged.cu", "split.cu", "abi.cu", "boys_device.cuh", "boys_eval.cuh"):
    src[fn] = open(f"paper_2504_07637_b200/csrc/{fn}").read().split("\n")
print(f"{len(insts)} SASS, {ti} warp-instr executed, {ts} stall samples")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -(kv[1][0] / ti + kv[1][1] / ts))[:int(sys.argv[5]) if len(sys.argv) > 5 else 30]:
    s = src.get(f, [""] * 100000)[ln - 1].strip()[:75] if f in src and ln else ""
    print(f"{100 * v[0] / ti:5.1f}% instr {100 * v[1] / ts:5.1f}% stall  {f}:{ln}  {s}")
