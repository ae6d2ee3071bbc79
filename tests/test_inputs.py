"""Pins of the seeded input generator (CPU only)."""
import os

import numpy as np

import ptdr_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    # Random123 kat_vectors (tests/golden/philox4x32_10_kat.txt)
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        ctr = [int(v, 16) for v in r[0:4]]
        key = [int(v, 16) for v in r[4:6]]
        want = tuple(int(v, 16) for v in r[6:10])
        assert ptdr_inputs.philox4x32_10(ctr, key) == want


def test_normal_moments():
    n = 8
    A = ptdr_inputs.dense(n, 1, "general")
    x = np.concatenate([A.real.ravel(), A.imag.ravel()])
    assert abs(x.mean()) < 0.01
    assert abs(x.var() - 1.0) < 0.02
    # real and imaginary parts independent
    assert abs(np.corrcoef(A.real.ravel(), A.imag.ravel())[0, 1]) < 0.01


def test_rows_are_consistent_slices():
    n = 6
    A = ptdr_inputs.dense(n, 0, "general")
    part = ptdr_inputs.dense(n, 0, "general", row0=17, nrows=9)
    assert np.array_equal(A[17:26], part)
    assert A[3, 5] == ptdr_inputs.entry(n, 0, 0, 3, 5)
    assert A[3, 5] == ptdr_inputs.normal_pair(0, 3 * 64 + 5, 0)


def test_hermitian_and_symmetric_are_exact():
    n = 6
    H = ptdr_inputs.dense(n, 2, "hermitian")
    assert np.array_equal(H, H.conj().T)
    assert np.all(np.diag(H).imag == 0)
    G = ptdr_inputs.dense(n, 2, "general")
    assert np.array_equal(H, (G + G.conj().T) / 2)  # A = (B + B^*)/2, same B
    S = ptdr_inputs.dense(n, 2, "real_symmetric")
    assert np.array_equal(S, S.T) and np.all(S.imag == 0)
    iu = np.triu_indices(1 << n)
    assert np.array_equal(S[iu], G.real[iu])


def test_band_layout():
    n = 5
    sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
    assert sub[0] == 0 and sup[-1] == 0
    assert np.array_equal(sub[1:], sup[:-1])         # symmetric
    assert np.all(main.imag == 0) and np.all(sup.imag == 0)
    d = ptdr_inputs.band(n, 3, "diagonal")
    assert d[4] == ptdr_inputs.normal_pair(3, 4, 1)
    assert main[4].real == d[4].real                  # same stream-1 draw, real part
