"""Developer: time decompose_batched (n, batch) with CUDA events (median of 10)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2403_11644_b200 as ptdr
from tools_bench_configs import time_it
n, B = int(sys.argv[1]), int(sys.argv[2])
A = torch.randn(B, 1 << n, 1 << n, dtype=torch.complex128, device="cuda")
out = torch.empty(B, 4 ** n, dtype=torch.complex128, device="cuda")
ms = time_it(lambda: ptdr.decompose_batched(A, out=out))
print(json.dumps({"n": n, "batch": B, "ms": ms, "alg_gbs": 32 * B * 4 ** n / ms / 1e6}))
