"""Static SASS census by outermost source line (nvdisasm -gi listing): instruction
counts of one function inside an address range, attributed to the line of the
top-level file (inlined callees fold into their call site).
usage: sass_static_lines.py listing.txt func_substr topfile lo hi"""
import re
import sys
from collections import Counter

txt, func, top, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4], 16), int(sys.argv[5], 16)
on, cur, agg, ops = False, None, Counter(), {}
for l in open(txt):
    if l.startswith(".text."):
        on = func in l
        continue
    if not on:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if m.group(1).endswith(top):
            cur = int(m.group(2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and lo <= int(m.group(1), 16) < hi:
        agg[cur] += 1
        op = m.group(2).split()[0] if not m.group(2).startswith("@") else m.group(2).split()[1]
        ops.setdefault(cur, Counter())[op.split(".")[0]] += 1
src = open(f"paper_2504_07637_b200/csrc/{top}").read().split("\n")
print(sum(agg.values()), "instructions")
for ln, c in sorted(agg.items(), key=lambda kv: kv[0] or 0):
    print(f"{c:5d}  {top}:{ln}  {src[ln - 1].strip()[:60] if ln else ''}   {dict(ops[ln].most_common(6))}")
