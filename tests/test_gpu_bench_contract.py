"""bench.py's own arm on the GPU honours the driver's JSON-line contract:
one line, the base keys, roofline / clocks / e2e / cpu_baseline / gpu_launches
with their sub-keys, and plausible values (short run, no extra configs)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_json_line_on_gpu():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "5", "--warmup", "3",
                        "--no-extras", "--e2e-steps", "1", "--cpu-seconds", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "clocks", "gpu_launches", "e2e", "cpu_baseline", "accuracy"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and "workload" in d["config"]
    ro = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in ro, k
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and 0.3 < ro["frac"] <= 1.0
    assert abs(ro["achieved"] / ro["peak"] - ro["frac"]) < 1e-3
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    # per step: the evaluator launch + the per-shard error reduction
    assert d["gpu_launches"] == 5 * 2 and d["gpu_launches_per_step"]["evaluator"] == 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * (1 << 26)
    assert e["d2h_bytes_per_step"] == 8 * 17 * (1 << 26)
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["max_ulp_gpu_vs_port"] == 0
    acc = d["accuracy"]
    assert acc["bits"] > 42.1 and len(acc["per_rank"]) == 1 and acc["max_ulp_vs_port"] == 0
