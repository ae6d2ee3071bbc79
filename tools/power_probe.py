"""Developer: board power and SM clock during long loops of (a) the n = 15 dense
decomposition, (b) a plain 16 GiB device copy at a similar byte rate (nvidia-smi, 50 ms)."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_11644_b200 as ptdr  # noqa: E402


def sample(fn, seconds=6.0):
    lines = []
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=power.draw,clocks.sm,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    t = threading.Thread(target=lambda: [lines.append(l.strip()) for l in p.stdout], daemon=True)
    t.start()
    t0 = time.time()
    n = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    p.terminate()
    t.join(timeout=2)
    vals = [l.split(",") for l in lines if l.count(",") == 2]
    pw = sorted(float(v[0]) for v in vals[len(vals) // 4:])
    ck = sorted(float(v[1]) for v in vals[len(vals) // 4:])
    cap = sum(1 for v in vals if "Active" in v[2]) / max(1, len(vals))
    return {"iters": n, "ms_per_iter": ev0.elapsed_time(ev1) / n, "power_w_median": pw[len(pw) // 2],
            "sm_mhz_median": ck[len(ck) // 2], "power_cap_frac": cap}


n = 15
A = ptdr.generate_dense(n, 4, "general")
out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, "general", 1, "cuda")
print("dense", sample(lambda: ptdr.decompose(A, "general", out=out, workspace=ws)), flush=True)
print("copy ", sample(lambda: out.copy_(A.view(-1))), flush=True)
