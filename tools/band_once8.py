"""Developer: one n=24 z-shard (rank 0 of 8) per tridiagonal structure, for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
n = 24
for structure in ("tridiagonal", "hermitian_tridiagonal"):
    B = ptdr.generate_band(n, 3, structure)
    for _ in range(2):
        ptdr.decompose_zshard(B, structure, 0, 8)
    torch.cuda.synchronize()
    del B
print("ok")
