"""Developer: one matrix-free decomposition (MODE_GEN) at n = 15 and the stored generator, timed."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from tools_bench_configs import time_it
n = 15
out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
ws = torch.empty(int(ptdr.lib().ptdr_generated_workspace_bytes(n, 1)), dtype=torch.uint8, device="cuda")
ms = time_it(lambda: ptdr.decompose_generated(n, 4, out=out, workspace=ws), iters=3, warm=1)
A = torch.empty((1 << n, 1 << n), dtype=torch.complex128, device="cuda")
gms = time_it(lambda: ptdr.generate_dense(n, 4, "general", out=A), iters=3, warm=1)
print(json.dumps({"matrix_free_ms": ms, "generator_ms": gms}))
