"""Host<->device copy rates for the e2e path: pinned 16 GiB H2D / D2H, allocation cost."""
import json, time, torch
n = 15
nb = 16 << (2 * n)
h = torch.empty(nb // 16, dtype=torch.complex128, pin_memory=True)
h2 = torch.empty(nb // 16, dtype=torch.complex128, pin_memory=True)
res = {}
t = time.perf_counter(); d = torch.empty(nb // 16, dtype=torch.complex128, device="cuda"); torch.cuda.synchronize(); res["alloc_s"] = time.perf_counter() - t
for it in range(2):
    t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); res["h2d_s"] = time.perf_counter() - t
    t = time.perf_counter(); h2.copy_(d, non_blocking=True); torch.cuda.synchronize(); res["d2h_s"] = time.perf_counter() - t
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); res["bidir_s"] = time.perf_counter() - t
res["h2d_gbs"] = nb / res["h2d_s"] / 1e9
res["d2h_gbs"] = nb / res["d2h_s"] / 1e9
res["bidir_gbs"] = 2 * nb / res["bidir_s"] / 1e9
print(json.dumps(res))
