# developer: look-ahead check of the dense pipeline -- default L vs the previous formula's L
cat > /tmp/herm_once.py <<'PY'
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
for cfg in "11 general 21" "12 general 11" "13 general 6" "14 general 3" "15 general 2" "16 general 2" "13 hermitian 11" "15 hermitian 3" "14 real_symmetric 6"; do
  set -- $cfg
  echo -n "$2$1 new "; timeout 120 python /tmp/herm_once.py $1 $2 2>&1 | tail -1
  echo -n "$2$1 old "; PTDR_L=$3 timeout 120 python /tmp/herm_once.py $1 $2 2>&1 | tail -1
done
done
