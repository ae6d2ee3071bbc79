"""Developer: under the power cap, does a capped persistent grid (fewer SMs at a higher
clock) move the n = 15 dense decomposition faster?  Sustained back-to-back loops (as the
bench), median ms per call and the SM clock / power sampled by nvidia-smi during each loop."""
import json, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_11644_b200 as ptdr

n = 15
A = ptdr.generate_dense(n, 4, "general")
out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, "general", 1)


def sample(stop, rec):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            c, p = r.stdout.strip().split(",")
            rec.append((float(c), float(p)))
        except ValueError:
            pass
        time.sleep(0.2)


for cap in [0, 144, 136, 128, 120, 112, 104, 96]:
    for _ in range(20):
        ptdr.decompose_xshard(A.view(-1), n, 0, 1, out=out, workspace=ws, max_ctas=cap)
    torch.cuda.synchronize()
    rec, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, rec))
    th.start()
    ts = []
    for _ in range(150):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ptdr.decompose_xshard(A.view(-1), n, 0, 1, out=out, workspace=ws, max_ctas=cap)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = [a.elapsed_time(b) for a, b in ts[50:]]
    print(json.dumps({"max_ctas": cap, "ms_median": float(np.median(ms)),
                      "sm_mhz_median": float(np.median([c for c, _ in rec])) if rec else None,
                      "power_w_median": float(np.median([p for _, p in rec])) if rec else None}), flush=True)
