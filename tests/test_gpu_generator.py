"""GPU generator kernel (row a1) vs the host input module (independent code).

Philox integers are identical by construction; the Box-Muller floats may differ
by a few ulp (CUDA vs glibc log/sincos), so the check is |d| <= 8 ulp-ish."""
import numpy as np
import pytest

import paper_2403_11644_b200 as ptdr
import ptdr_inputs

pytestmark = pytest.mark.gpu


def _close(a, b):
    return np.max(np.abs(a - b)) <= 4e-15 * max(1.0, np.max(np.abs(b)))


@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_dense_generator_matches_host(gpu, variant):
    n = 9
    got = ptdr.generate_dense(n, 4, variant).cpu().numpy()
    want = ptdr_inputs.dense(n, 4, variant)
    assert _close(got, want)
    if variant == "hermitian":
        assert np.array_equal(got, got.conj().T)       # exact on the device too
    part = ptdr.generate_dense(n, 4, variant, row0=100, nrows=7).cpu().numpy()
    assert np.array_equal(part, got[100:107])          # row split does not change values


def test_band_generator_matches_host(gpu):
    n = 12
    got = ptdr.generate_band(n, 3, "tridiagonal").cpu().numpy()
    sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
    assert _close(got, np.stack([sub, main, sup]))
    d = ptdr.generate_band(n, 3, "diagonal").cpu().numpy()
    assert _close(d, ptdr_inputs.band(n, 3, "diagonal"))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sendblocks_layout(gpu, world):
    n = 8
    N, R = 1 << n, (1 << n) // world
    A = ptdr.generate_dense(n, 4, "general").cpu().numpy()
    for rank in range(world):
        s = ptdr.generate_sendblocks(n, 4, rank, world).cpu().numpy()
        for b in range(world):
            want = A[rank * R:(rank + 1) * R, (rank ^ b) * R:((rank ^ b) + 1) * R]
            assert np.array_equal(s[b], want)
