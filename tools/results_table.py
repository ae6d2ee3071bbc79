"""Markdown table of a tools_bench_configs.py JSONL file (for DESIGN.md section 11)."""
import json, sys

rows = []
for line in open(sys.argv[1]):
    try:
        d = json.loads(line)
    except ValueError:
        continue
    if "config" not in d:
        continue
    ms = d.get("ms", d.get("ms_per_rank"))
    if ms is None:
        continue
    cps = d.get("coeffs_per_s", d.get("coeffs_per_s_total"))
    frac = d.get("frac_of_measured", d.get("frac_of_measured_16B"))
    orc = d.get("oracle_coeffs_per_s")
    g = d.get("graph_replay_ms")
    rows.append(f"| {d['config']} | {ms:.4g} | {'' if g is None else f'{g:.3g}'} | {cps:.3g} | "
                f"{'' if frac is None else f'{frac:.2f}'} | {'' if orc is None else f'{orc:.3g}'} |")
print("| config | ms | graph-replay ms | coeffs/s | frac of measured HBM | oracle coeffs/s (16 cores) |")
print("|---|---|---|---|---|---|")
print("\n".join(rows))
