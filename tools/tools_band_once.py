import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
v = sys.argv[1] if len(sys.argv) > 1 else "tridiagonal"
n = 24
B = ptdr.generate_band(n, 3, v, device="cuda")
out = torch.empty(ptdr.output_count(n, v), dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, v, 1, "cuda")
for _ in range(3):
    ptdr.decompose(B, v, out=out, workspace=ws)
torch.cuda.synchronize()
print("ok")
