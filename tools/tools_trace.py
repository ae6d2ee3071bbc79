"""Run one n=15 decomposition with PTDR_TRACE=1 and print the CTA-0 pipeline timeline."""
import ctypes, os, sys
os.environ["PTDR_TRACE"] = "1"
os.environ["PTDR_LIB_NAME"] = "libptdr_trace.so"   # build with PTDR_TRACE_BUILD=1
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_11644_b200 as ptdr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
A = ptdr.generate_dense(n, 4, "general", device="cuda")
out = torch.empty(1 << (2 * n), dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, "general", 1, "cuda")
for _ in range(3):
    ptdr.decompose(A, out=out, workspace=ws)
torch.cuda.synchronize()
L = ptdr.lib()
L.ptdr_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros(512 * 16, dtype=np.uint64)
r = L.ptdr_debug_trace_copy(buf.ctypes.data, buf.nbytes)
t = buf.reshape(512, 16).astype(np.int64)
valid = t[:, 1] > 0
t0 = t[valid][:, 0].min()
np.save("gpurun_out/trace.npy", t)
print("k phase | prod: wait_empty dep issue | cons: wait meta/full ready->release release->done | (cycles rel.)")
for k in range(0, 400):
    r = t[k]
    if r[1] == 0: continue
    print(k, r[8], "|", r[1]-r[0], r[2]-r[1], r[3]-r[2], "|", r[5]-r[4], r[6]-r[5], r[7]-r[6], "| issue@", r[3]-t0, "ready@", r[5]-t0, "done@", r[7]-t0)
