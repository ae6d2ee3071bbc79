"""Time the n=15 dense decomposition with the library named by PTDR_LIB_NAME (diagnostic
builds: libptdr_diag1.so = no output stores, libptdr_diag2.so = L2-resident phase-A loads)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
from tools_bench_configs import time_it  # noqa
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
A = ptdr.generate_dense(n, 4, "general", device="cuda")
out = torch.empty(1 << (2 * n), dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, "general", 1, "cuda")
ms = time_it(lambda: ptdr.decompose(A, "general", out=out, workspace=ws))
print(json.dumps({"lib": os.environ.get("PTDR_LIB_NAME", "libptdr.so"), "n": n, "ms": ms,
                  "alg_gbs": 32 * 4**n / ms / 1e6}))
