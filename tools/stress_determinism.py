"""Developer: repeat the dense decomposition many times and require bitwise-identical outputs
(the pipeline's arithmetic order is fixed, so any mismatch would expose a race in the
inter-CTA hand-off).  usage: stress_determinism.py [reps_small] [reps_large]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr

reps_small = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps_large = int(sys.argv[2]) if len(sys.argv) > 2 else 20
res = {}
t0 = time.time()
for n, variant, reps in [(11, "general", reps_small), (12, "general", reps_small), (13, "hermitian", reps_small),
                         (14, "real_symmetric", reps_large), (15, "general", reps_large)]:
    A = ptdr.generate_dense(n, 4, variant)
    ws = ptdr.alloc_workspace(n, variant, 1, "cuda")
    ref = ptdr.decompose(A, variant, workspace=ws).clone()
    out = torch.empty_like(ref)
    bad = 0
    for _ in range(reps):
        out.fill_(float("nan"))
        ptdr.decompose(A, variant, out=out, workspace=ws)
        if not torch.equal(torch.view_as_real(out).view(torch.int64), torch.view_as_real(ref).view(torch.int64)):
            bad += 1
    torch.cuda.synchronize()
    res[f"n{n}_{variant}"] = {"reps": reps, "mismatches": bad}
    del A, ws, ref, out
    torch.cuda.empty_cache()
# the inverse on the pipeline (q order and matrix layout), the tail pipeline (n = 24 diagonal)
# and the fused tridiagonal expansion (both tridiagonal structures)
for n, reps in [(12, reps_small), (15, reps_large)]:
    c = ptdr.decompose(ptdr.generate_dense(n, 4, "general"))
    ref = ptdr.reconstruct(c).clone()
    out = torch.empty_like(ref)
    bad = 0
    for _ in range(reps):
        out.fill_(float("nan"))
        ptdr.reconstruct(c, out=out)
        bad += 0 if torch.equal(torch.view_as_real(out).view(torch.int64), torch.view_as_real(ref).view(torch.int64)) else 1
    res[f"n{n}_inverse_q"] = {"reps": reps, "mismatches": bad}
    del c, ref, out
    torch.cuda.empty_cache()
for structure in ("diagonal", "tridiagonal", "hermitian_tridiagonal"):
    B = ptdr.generate_band(24, 3, structure)
    ref = ptdr.decompose(B, structure).clone()
    out = torch.empty_like(ref)
    bad = 0
    for _ in range(reps_large):
        out.fill_(float("nan"))
        ptdr.decompose(B, structure, out=out)
        bad += 0 if torch.equal(torch.view_as_real(out).view(torch.int64), torch.view_as_real(ref).view(torch.int64)) else 1
    res[f"n24_{structure}"] = {"reps": reps_large, "mismatches": bad}
    del B, ref, out
    torch.cuda.empty_cache()
res["seconds"] = round(time.time() - t0, 1)
print(json.dumps(res))
assert all(v["mismatches"] == 0 for k, v in res.items() if k != "seconds"), res
