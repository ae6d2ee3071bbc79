"""Time the dense generator kernel (row a1) at n=15: write-bound roofline 16 B/element."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
from tools_bench_configs import time_it, PEAK
n = 15
A = torch.empty((1 << n, 1 << n), dtype=torch.complex128, device="cuda")
ms = time_it(lambda: ptdr.generate_dense(n, 4, "general", out=A), iters=5, warm=2)
print(json.dumps({"kernel": "gen_dense_kernel", "n": n, "ms": ms, "gbs": 16 * 4 ** n / ms / 1e6,
                  "frac_of_measured": 16 * 4 ** n / ms / 1e6 / PEAK}))
