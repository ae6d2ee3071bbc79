"""Developer: host-side cost of one decomposition call at small n (the configs[0]/[1] sizes are
launch-bound).  Times 2000 back-to-back calls (device work queued asynchronously) through
(a) the Python binding and (b) the raw C ABI via ctypes with pre-built arguments, and the
device time of one call from CUDA events.  usage: host_overhead.py n"""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_11644_b200 as ptdr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
A = ptdr.generate_dense(n, 0, "general")
out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, "general", 1, "cuda")
for _ in range(50):
    ptdr.decompose(A, out=out, workspace=ws)
torch.cuda.synchronize()
K = 2000
t0 = time.perf_counter()
for _ in range(K):
    ptdr.decompose(A, out=out, workspace=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
lib = ptdr.lib()
args = (ctypes.c_void_p(A.data_ptr()), n, 0, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
        ctypes.c_size_t(ws.numel()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
f = lib.ptdr_decompose_async
t3 = time.perf_counter()
for _ in range(K):
    f(*args)
t4 = time.perf_counter()
torch.cuda.synchronize()
t5 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    f(*args)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"n": n, "binding_us_per_call": (t1 - t0) / K * 1e6, "binding_wall_us": (t2 - t0) / K * 1e6,
                  "cabi_us_per_call": (t4 - t3) / K * 1e6, "cabi_wall_us": (t5 - t3) / K * 1e6,
                  "device_us_per_call_queued": e0.elapsed_time(e1) / 100 * 1e3}))
