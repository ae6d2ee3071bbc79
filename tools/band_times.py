"""Developer timing of the structured paths at n = 24 (BASELINE configs[3]): one GPU and the
per-rank z-shard at G = 2 / 4 / 8 (ranks are independent; max over the ranks timed), CUDA
events, median of 10.  Algorithmic bytes per rank: band read (the
whole band: every rank reads it) + the rank's output."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_11644_b200 as ptdr  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from tools_bench_configs import PEAK, time_it  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
for structure in ("diagonal", "anti_diagonal", "tridiagonal", "hermitian_tridiagonal"):
    B = ptdr.generate_band(n, 3, "diagonal" if structure == "anti_diagonal" else structure)
    blocks = n + 1 if "tridiagonal" in structure else 1
    for world in (1, 2, 4, 8):
        NL = (1 << n) // world
        outl = torch.empty(blocks * NL, dtype=torch.complex128, device="cuda")
        ws = ptdr.alloc_workspace(n, structure, world, "cuda")
        ranks = [0] if world == 1 else sorted({0, world // 2, world - 1})
        ms = max(time_it(lambda r=r: ptdr.decompose_zshard(B, structure, r, world, out=outl, workspace=ws))
                 for r in ranks)
        alg = B.numel() * 16 + outl.numel() * 16
        print(json.dumps({"n": n, "structure": structure, "world": world, "ms_per_rank": ms,
                          "alg_bytes_per_rank": alg, "frac": alg / (ms * 1e-3) / 1e9 / PEAK}), flush=True)
        del outl, ws
    del B
    torch.cuda.empty_cache()
