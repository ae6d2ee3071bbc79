"""Developer: time ptdr.reconstruct_matrix_layout (out of place) at n (CUDA events, median of 10)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_11644_b200 as ptdr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
N = 1 << n
M = torch.randn((N, N), dtype=torch.complex128, device="cuda")
out = torch.empty((N, N), dtype=torch.complex128, device="cuda")
ws = torch.empty(int(ptdr.lib().ptdr_reconstruct_matrix_layout_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ptdr.reconstruct_matrix_layout(M, out=out, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"n": n, "ms": float(np.median(ts))}))
