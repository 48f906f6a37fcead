"""cfg1 as a stream of 32 distinct 2^20-point batches replayed from one CUDA
graph (the bench's cfg1 line), repeated: prints per-launch microseconds."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
from paper_2504_07637_b200 import _lib  # noqa: E402

_lib.load(build_if_missing=False)
dev = torch.device("cuda:0")
res = {}
for name, rot in (("cfg1", 32), ("cfg2", 1), ("cfg3", 1)):
    wl = B.make_workload(name, 0, 1, dev, rotate=rot)
    steps = 100 if name == "cfg1" else 20
    secs, per, _, n = B.time_workload(wl, steps, 5, 1, 0, graph=(rot > 1))
    res[name] = {"us_per_launch": round(1e3 * sum(per) / len(per), 3),
                 "job_us_per_launch": round(1e6 * secs / (steps * rot), 3)}
    del wl
    torch.cuda.empty_cache()
print(json.dumps({"pdl": os.environ.get("BOYS_PDL", "1"), **res}))
