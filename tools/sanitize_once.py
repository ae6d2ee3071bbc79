"""Small runs of every kernel family, for compute-sanitizer (one tool per process).

    compute-sanitizer --tool memcheck python tools/sanitize_once.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr

dev = torch.device("cuda:0")
for n in (4, 6, 9, 11):
    for v in ("general", "hermitian", "real_symmetric"):
        A = ptdr.generate_dense(n, 1, v, device=dev)
        ptdr.decompose(A, v)
for v in ("diagonal", "tridiagonal"):
    B = ptdr.generate_band(12, 3, v, device=dev)
    ptdr.decompose(B, v)
    ptdr.decompose_zshard(B, v, 1, 4)
ptdr.decompose(ptdr.generate_band(12, 3, "diagonal", device=dev), "anti_diagonal")
g = torch.Generator(device="cuda").manual_seed(1)
d = torch.complex(torch.randn(5, 1 << 10, generator=g, device="cuda", dtype=torch.float64),
                  torch.randn(5, 1 << 10, generator=g, device="cuda", dtype=torch.float64))
ptdr.decompose_band(d, 2)
A = ptdr.generate_dense(9, 2, "general", device=dev)
c = ptdr.decompose(A)
ptdr.reconstruct(c)
ptdr.reconstruct(ptdr.decompose(ptdr.generate_dense(6, 2, "general", device=dev)))
ptdr.axpby(1.0, c, 2.0, c)
ptdr.direct_sum(c, c)
ptdr.hermitian_augment(c)
ptdr.decompose_batched(torch.randn((3, 64, 64), dtype=torch.complex128, device=dev))
ptdr.decompose_padded(torch.randn((100, 100), dtype=torch.complex128, device=dev))
ptdr.coefficients(A, torch.arange(0, 4 ** 9, 997, device=dev))
ptdr.decompose_generated(11, 4)
R = (1 << 11) // 2
shards = [ptdr.generate_dense(11, 4, "general", row0=r * R, nrows=R, device=dev) for r in range(2)]
ptdr.decompose_peer([s.data_ptr() for s in shards], 11, 0, 2)
torch.cuda.synchronize()
print("sanitize_once ok")
