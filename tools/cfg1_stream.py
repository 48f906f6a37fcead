"""cfg1 timed the two ways bench.py reports it: (a) a stream of 32 distinct
2^20-point batches replayed from one CUDA graph, (b) one batch with L2 flushed
before every launch; plus cfg2/cfg3 single launches.  Prints one JSON line of
per-launch microseconds (the kernel variant is chosen by the environment)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402

ctx = B.Ctx()
flushbuf = torch.empty(1 << 30, dtype=torch.uint8, device=ctx.dev)
res = {"env": {k: v for k, v in os.environ.items() if k.startswith("BOYS_")}}
for key, name, rot, mode in (("cfg1", "cfg1", 32, "graph"), ("cfg1_l2flush", "cfg1", 1, "flush"),
                             ("cfg2", "cfg2", 1, None)):
    wl = B.make_workload(name, ctx, rotate=rot)
    steps = 100 if rot > 1 else 200
    r = B.time_workload(wl, ctx, steps, 5, flush=(lambda: flushbuf.zero_()) if mode == "flush" else None,
                        graph=mode == "graph")
    per = r["per_launch_ms"]
    res[key] = {"us_per_launch": round(1e3 * sum(per) / len(per), 3)}
    del wl
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
