"""One dense decomposition (for ncu launch lists): tools/dense_once.py n variant"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
n, v = int(sys.argv[1]), sys.argv[2]
A = ptdr.generate_dense(n, 2, v)
out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, v, 1, "cuda")
for _ in range(3):
    ptdr.decompose(A, v, out=out, workspace=ws)
torch.cuda.synchronize()
print("ok")
