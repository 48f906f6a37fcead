"""bench.py's own multi-rank plumbing on CPU: `--gpus 2` outside torchrun
re-executes under torch.distributed.run with two ranks (gloo in the CPU
self-test), and the timing (barrier -> steps -> error gather -> barrier,
max over ranks), the value sum and the per-rank error gather come from the
same functions the GPU arm uses (Ctx, time_workload, accuracy_obj); only the
evaluator is a CPU stub."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(gpus):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--stub", "--gpus", str(gpus),
                        "--steps", "4", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_gloo():
    d = _run(2)
    assert d["n_gpus"] == 2 and d["steps"] == 4
    secs, vals = d["per_rank"]["secs"], d["per_rank"]["values"]
    assert len(secs) == 2 and len(vals) == 2 and all(s > 0 for s in secs)
    # job time = max over ranks; value = all ranks' values / job time
    assert abs(d["ms_per_step"] * d["steps"] / 1e3 - max(secs)) <= 1e-9 * max(secs) + 1e-12
    assert abs(d["value"] - sum(vals) / max(secs)) <= 1e-6 * d["value"]
    acc = d["accuracy"]
    assert len(acc["per_rank"]) == 2 and acc["max_rel_err"] == max(acc["per_rank"])
    assert acc["max_rel_err"] < 1e-15


def test_bench_one_rank_no_torchrun():
    d = _run(1)
    assert d["n_gpus"] == 1 and len(d["per_rank"]["secs"]) == 1
