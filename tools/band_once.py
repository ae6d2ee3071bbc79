"""One n=24 structured decomposition per configuration (for ncu launch lists): diagonal and
tridiagonal on one GPU, and rank 0 of their z-shards at G = 8."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_11644_b200 as ptdr  # noqa: E402

n = 24
for structure in ("diagonal", "tridiagonal"):
    B = ptdr.generate_band(n, 3, structure)
    for world in (1, 8):
        for _ in range(2):
            ptdr.decompose_zshard(B, structure, 0, world)
    torch.cuda.synchronize()
    del B
print("ok")
