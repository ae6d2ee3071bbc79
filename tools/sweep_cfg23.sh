# developer: configurations 1, 2, 3 (16-wide chunks; 64 KiB tiles x 2 groups vs 32 KiB tiles x
# 4 / 3 groups) at n = 15 / 16, dev library
export PTDR_LIB_NAME=libptdr_dev.so
cat > /tmp/var_once.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_2403_11644_b200 as ptdr
from tools_bench_configs import time_it
n = int(sys.argv[1]); v = sys.argv[2]
A = ptdr.generate_dense(n, 2, v)
out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
ws = ptdr.alloc_workspace(n, v, 1, "cuda")
print(json.dumps({"ms": time_it(lambda: ptdr.decompose(A, v, out=out, workspace=ws))}))
PY
for r in 1 2; do
for cfg in "15 general" "13 general"; do
  set -- $cfg
  for C in 1 2 3; do echo -n "$2$1 cfg=$C "; PTDR_PIPE_CFG=$C timeout 120 python /tmp/var_once.py $1 $2 2>&1 | tail -1; done
done
done
