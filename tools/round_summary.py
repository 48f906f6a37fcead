"""One-page round summary (markdown on stdout) from the committed evidence:
profiles/rNN_bench.jsonl, rNN_bench_reference.jsonl, rNN_ncu_raw.csv, ncu_traffic.json.
usage: python tools/round_summary.py r02 > profiles/r02_summary.md"""
import csv
import json
import sys
from pathlib import Path

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
P = Path(__file__).resolve().parents[1] / "profiles"


def last_json(path):
    return [json.loads(l) for l in open(path) if l.startswith("{")][-1]


b = last_json(P / f"{tag}_bench.jsonl")
refs = [json.loads(l) for l in open(P / f"{tag}_bench_reference.jsonl") if l.startswith("{")]
ref = next(r for r in refs if r.get("impl") == "reference")
ncu = {}
rows = list(csv.reader(open(P / f"{tag}_ncu_raw.csv")))
hdr = rows[0]
ki, di = hdr.index("Kernel Name"), hdr.index("gpu__time_duration.sum")
for r in rows[2:]:
    if len(r) == len(hdr):
        ncu.setdefault(r[ki], []).append(float(r[di].replace(",", "")))
unit = rows[1][di]


def ncu_ms(sub):
    for k, v in ncu.items():
        if sub in k:
            d = v[-1]
            return d / 1e3 if unit in ("us", "usecond") else (d / 1e6 if unit in ("ns", "nsecond") else d)
    return None


ALG = "algorithmic_bytes_per_launch"
KER = {"cfg3": "dense_kernel<double, 16", "cfg1": "dense_soa_quad0_spec_kernel<double", "cfg2": "dense_soa_pair_kernel<double, 8",
       "cfg4": "ragged_kernel<double", "cfg4f32": "ragged_kernel<float", "cfg5": "dense_kernel<double, 12",
       "split": "split_kernel<double, 16", "hermite": "hermite_kernel<4>"}
rf, ck = b["roofline"], b["clocks"]
print(f"# Round summary {tag} (one B200; `profiles/{tag}_bench.jsonl`, `{tag}_ncu_summary.md`)\n")
print(f"Headline: {b['config']['workload']} -- **{b['value'] / 1e9:.1f}e9 F-values/s**, {b['ms_per_step']:.4f} ms per step, "
      f"**{100 * rf['frac']:.1f}% of the measured HBM copy bandwidth** ({rf['achieved']:.0f} of {rf['peak']} GB/s), DRAM traffic "
      f"{rf['traffic'] / rf['algorithmic_bytes_per_launch']:.3f} x algorithmic; clocks median {ck['sm_mhz']} MHz ({', '.join(ck['reasons']) or 'no throttle reason'}). "
      f"Accuracy vs refmath goldens on the timed outputs: {b['accuracy']['bits']:.2f} bits; {b['accuracy']['max_ulp_vs_port']:.0f} ulp vs the CPU restatement.\n")
print("| config | value | per launch (events) | ncu duration | roofline | DRAM / algorithmic | accuracy (bits vs refmath / ulp vs port) |")
print("|---|---|---|---|---|---|---|")


def line(name, e):
    r = e["roofline"]
    n = ncu_ms(KER.get(name.split("_")[0], "?"))
    tr = r.get("traffic")
    a = e.get("accuracy", {})
    acc = f"{a['bits']:.1f} / {a.get('max_ulp_vs_port', 0):.0f}" if "bits" in a else "-"
    print(f"| {name} | {e['value'] / 1e9:.1f}e9 {e['unit']} | {r['launch_ms']:.4f} ms | {f'{n:.4f} ms' if n and name in KER else '-'} | "
          f"{100 * r['frac']:.1f}% {'FP64' if r['bound'] == 'fp64' else 'HBM'} | {f'{tr / r[ALG]:.3f}' if tr else '-'} | {acc} |")


line("cfg3", b)
for k, e in b.get("configs", {}).items():
    if "roofline" in e:
        line(k, e)
c4, c4f = b["configs"].get("cfg4", {}), b["configs"].get("cfg4f32", {})
print(f"\nOffsets scan ({c4.get('offsets_elements', 0)} orders): {c4.get('offsets_ms')} ms, bit-identical: {c4.get('offsets_bit_identical')}. "
      f"End to end (cfg3, pinned host buffers through `boys_eval_dense_host`): {b['e2e']['value'] / 1e9:.2f}e9 values/s "
      f"(PCIe D2H-bound: {b['e2e']['d2h_bytes_per_step'] / 1e9:.1f} GB of results per step); cfg4 e2e "
      f"{c4.get('e2e', {}).get('value', 0) / 1e9:.2f}e9 values/s.\n")
cb, cr = b["cpu_baseline"], b.get("cpu_baseline_reference", {})
print(f"CPU baselines on the box's {cb['cores']} host threads ({cb.get('cpu_model', '?')}): the C restatement {cb['value'] / 1e9:.2f}e9 values/s; "
      f"the reference's own `refmath.boys_downward` (mpmath, `baseline/_ref`) {cr.get('value', 0):.3g} values/s ({cr.get('sample', '')}). "
      f"Reference arm (`--impl reference`, {ref['cpu_baseline']['sample']}): {ref['value'] / 1e9:.2f}e9 values/s.\n")
if b.get("fp64_peak_measured_ops_per_s"):
    print(f"FP64 peak for the n=0 roofline: measured live by the DFMA probe, {b['fp64_peak_measured_ops_per_s'] / 1e12:.2f} T ops/s.")
