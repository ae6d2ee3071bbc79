"""The CPU oracle's per-core rate ("a single-thread n10 run"): run with
OMP_NUM_THREADS=1; coefficients/s of the explicit-string trace on seeded random strings of the
n = 10 general matrix (seed 1), bounded to ~3 s."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
import ptdr_inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
A = ptdr_inputs.dense(n, 1, "general")
rng = np.random.default_rng(11)
done, t0 = 0, time.perf_counter()
while time.perf_counter() - t0 < 3.0:
    oracle.coeffs_dense(A, rng.integers(0, 4 ** n, 64, dtype=np.uint64))
    done += 64
rate = done / (time.perf_counter() - t0)
print(json.dumps({"n": n, "oracle_threads": oracle.threads(), "oracle_coeffs_per_s_per_core": rate,
                  "full_decomposition_s_one_core": 4 ** n / rate}))
