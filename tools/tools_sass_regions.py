"""Summarise ncu source-page stall samples by SASS region (dev tool)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; idx = {n: i for i, n in enumerate(h)}; data = rows[2:]
reasons = ['stall_barrier','stall_long_sb','stall_short_sb','stall_wait','stall_selected','stall_not_selected','stall_mio','stall_lg','stall_math','stall_branch_resolving','stall_membar','stall_sleep','stall_no_inst','stall_dispatch']
def f(r, k):
    try: return float(r[idx[k]] or 0)
    except: return 0.0
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
# print per-instruction with cumulative, mark big ones
cum = {k: 0.0 for k in reasons}
for r in data:
    for k in reasons: cum[k] += f(r, k)
print('total', tot)
for k in reasons: print(f'{k:28s} {cum[k]/tot*100:6.2f}%')
if len(sys.argv) > 2:
    lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
    s = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data if lo <= int(r[idx['Address']], 16) <= hi)
    print('region', s / tot * 100)
