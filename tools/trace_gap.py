"""Producer timeline breakdown from gpurun_out/trace.npy (tools_trace.py output)."""
import numpy as np
t = np.load("gpurun_out/trace.npy").astype(np.int64)
ks = [k for k in range(40, 500) if t[k][1] > 0 and t[k + 1][0] > 0]
f = lambda a, b: np.mean([t[k][b] - t[k][a] for k in ks])
print("cycle", np.mean([t[k + 1][0] - t[k][0] for k in ks]))
print("wait_empty", f(0, 1), "dep", f(1, 2), "issue", f(2, 3), "3->9 (return+decode)", f(3, 9),
      "9->next0", np.mean([t[k + 1][0] - t[k][9] for k in ks]))
odd = [k for k in ks if t[k][10] > 0]
print("atomic stamp present on", len(odd), "tiles; 9->10", np.mean([t[k][10] - t[k][9] for k in odd]) if odd else None)
