"""One run of each 'next' path at a measurable size (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr
which = sys.argv[1]
if which == "band_s2":
    g = torch.Generator(device="cuda").manual_seed(5)
    d = torch.complex(torch.randn(5, 1 << 24, generator=g, device="cuda", dtype=torch.float64),
                      torch.randn(5, 1 << 24, generator=g, device="cuda", dtype=torch.float64))
    for _ in range(2):
        ptdr.decompose_band(d, 2)
elif which == "inverse":
    A = ptdr.generate_dense(15, 4, "general")
    c = ptdr.decompose(A)
    del A
    for _ in range(2):
        ptdr.reconstruct(c)
elif which == "matrix_free":
    for _ in range(2):
        ptdr.decompose_generated(15, 4)
torch.cuda.synchronize()
print("ok")
