"""gpurun_out/order_sweep.txt (tools/order_sweep.sh) -> profiles/r01_order_sweep.md."""
import json
import os
import sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))) + "/"
sys.path.insert(0, R)
from paper_2504_07637_b200 import roofline as RL  # noqa: E402

peak = json.load(open(R + "MEASURED_PEAKS.json"))["hbm_gbs"]
fp64 = 17.06e12
rows = {}
for line in open(R + "gpurun_out/order_sweep.txt"):
    dt, lay, js = line.split(" ", 2)
    for k, v in json.loads(js).items():
        if k.startswith("n"):
            rows.setdefault((dt, lay), {})[int(k.split("_")[0][1:])] = v
N = 1 << 24
L = ["# Order sweep: every (dtype, layout, order) at 2^24 points, default kernel choices", "",
     "`tools/order_sweep.sh` (graph-replayed stream of distinct batches, `tools/grid_rule.py`), one B200.",
     f"Fraction = algorithmic bytes (x + outputs) / time / {peak} GB/s (MEASURED_PEAKS.json copy peak);",
     "for the FP64-bound small f64 orders the FP64 fraction (algorithmic ops, 17.06 T DFMA/s probe) too.", "",
     "| n | f64 SoA µs | f64 SoA HBM | f64 AoS µs | f64 AoS HBM | f32 SoA µs | f32 SoA HBM | f32 AoS µs | f32 AoS HBM |",
     "|---|---|---|---|---|---|---|---|---|"]
for n in sorted({n for d in rows.values() for n in d}):
    cells = []
    for dt, lay in (("f64", "soa"), ("f64", "aos"), ("f32", "soa"), ("f32", "aos")):
        t = rows.get((dt, lay), {}).get(n)
        if t is None:
            cells += ["-", "-"]
            continue
        eb = 8 if dt == "f64" else 4
        frac = (eb + eb * (n + 1)) * N / (t * 1e-6) / 1e9 / peak
        extra = ""
        if dt == "f64" and n <= 3:
            extra = f" (FP64 {RL.ops_per_point(n) * N / (t * 1e-6) / fp64 * 100:.0f}%)"
        cells += [f"{t:.1f}", f"{frac * 100:.0f}%{extra}"]
    L.append(f"| {n} | " + " | ".join(cells) + " |")
L += ["", "Kernels (defaults): SoA n ≤ 3 four points per thread, else two (one block per tile; f32 n < 6",
      "persistent); AoS n = 0 → the SoA kernel, n = 1 (and f32 n = 3) register rows with direct 16-byte",
      "stores, f64 n ≤ 8 / all f32 two points per thread with staged bulk copies, f64 n ≥ 9 one point",
      "per thread with double-buffered staging."]
open(R + "profiles/r01_order_sweep.md", "w").write("\n".join(L) + "\n")
print("\n".join(L))
