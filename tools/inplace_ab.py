"""Developer: q-order out-of-place vs in-place, each call right after regenerating A."""
import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2403_11644_b200 as ptdr
for n in (15, 16):
    A = ptdr.generate_dense(n, 4, "general")
    ws_ip = torch.empty(int(ptdr.lib().ptdr_inplace_workspace_bytes(n, 0)), dtype=torch.uint8, device="cuda")
    out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
    ws = ptdr.alloc_workspace(n, "general", 1, "cuda")
    def run(kind):
        t = []
        for it in range(8):
            ptdr.generate_dense(n, 4, "general", out=A)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "inplace":
                ptdr.decompose(A, "general", workspace=ws_ip, inplace=True)
            else:
                ptdr.decompose(A, "general", out=out, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                t.append(e0.elapsed_time(e1))
        return sorted(t)[len(t) // 2]
    for rep in range(2):
        print(json.dumps({"n": n, "qorder_after_gen": run("q"), "inplace_after_gen": run("inplace")}), flush=True)
    del A, out, ws, ws_ip
    torch.cuda.empty_cache()
