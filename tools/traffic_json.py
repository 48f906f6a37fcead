"""ncu --set full report of tools/prof_kernels.py (configs in the given order,
--launches 2) -> profiles/ncu_traffic.json: DRAM read + write bytes per launch
of each config's kernel, from its SECOND launch (the first is cold).

    python tools/traffic_json.py REPORT.ncu-rep cfg3,cfg2,cfg1,cfg4,cfg4f32,cfg5,split SOURCE_NOTE
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, order, note = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki = hdr.index("Kernel Name")
rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = []
for r in rows[2:]:
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    launches.append((r[ki].split("(")[0], b))
res = {"source": note}
assert len(launches) == 2 * len(order), (len(launches), order)
for k, cfg in enumerate(order):
    name, b = launches[2 * k + 1]
    res[cfg] = int(round(b))
    res.setdefault("kernels", {})[cfg] = name
Path(__file__).resolve().parents[1].joinpath("profiles", "ncu_traffic.json").write_text(
    json.dumps(res, indent=1) + "\n")
print(json.dumps(res, indent=1))
