"""Independent dense Pauli construction for pins (numpy Kronecker products only).

The 2x2 matrices are retyped from PAPER.md l.37-55.  The tensor product is
numpy.kron with the leftmost text letter as the first (most significant)
factor, "P = sigma_{n-1} (x) ... (x) sigma_0".  Nothing here
uses the oracle's PauliComposer or the GPU path's XOR-mask identity.
"""
from functools import reduce

import numpy as np

PAULI = {
    "I": np.array([[1, 0], [0, 1]], dtype=np.complex128),
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "Z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
}
LETTERS = "IXYZ"


def all_strings(n):
    """Strings in ascending text-lexicographic order (I<X<Y<Z)."""
    if n == 0:
        return [""]
    return [a + s for a in LETTERS for s in all_strings(n - 1)]


def kron_string(text):
    return reduce(np.kron, [PAULI[c] for c in text])


def brute_force_coeffs(A):
    """alpha_P = Tr(P A)/2^n for every string, dense O(16^n)."""
    N = A.shape[0]
    n = N.bit_length() - 1
    return np.array([np.trace(kron_string(s) @ A) / N for s in all_strings(n)])


def reconstruct(coeffs, n):
    return sum(c * kron_string(s) for c, s in zip(coeffs, all_strings(n)))


def random_complex(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
