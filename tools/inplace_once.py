"""One n=15 in-place decomposition after warm-up (for ncu): tools/inplace_once.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
A = ptdr.generate_dense(n, 4, "general")
ws = torch.empty(int(ptdr.lib().ptdr_inplace_workspace_bytes(n, 0)), dtype=torch.uint8, device="cuda")
for _ in range(4):
    ptdr.generate_dense(n, 4, "general", out=A)
    ptdr.decompose(A, "general", workspace=ws, inplace=True)
torch.cuda.synchronize()
print("ok")
