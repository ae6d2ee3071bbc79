"""Developer: time decompose_band at (n, s) (CUDA events, median of 10) and leave one more
call for a profiler launch list.  usage: band_s_once.py n s [reps]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_11644_b200 as ptdr

n, s = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
N = 1 << n
g = torch.Generator(device="cuda").manual_seed(5)
d = torch.randn(2 * s + 1, N, dtype=torch.complex128, device="cuda", generator=g)
cnt = len(ptdr.band_xmasks(n, s))
out = torch.empty(cnt * N, dtype=torch.complex128, device="cuda")
ws = torch.empty(int(ptdr.lib().ptdr_band_workspace_bytes(n, s)), dtype=torch.uint8, device="cuda")
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ptdr.decompose_band(d, s, out=out, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
alg = (2 * s + 1) * N * 16 + cnt * N * 16
print(json.dumps({"n": n, "s": s, "blocks": cnt, "ms": ms, "alg_gbs": alg / ms / 1e6}))
