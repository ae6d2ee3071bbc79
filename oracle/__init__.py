"""CPU oracle for the Pauli decomposition -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path never does.

The arithmetic lives in oracle.c (plain C, OpenMP): the definition
alpha_P = Tr(P A)/2^n per coefficient, with P built explicitly
by PauliComposer (l.199-208) and the trace of Algorithm 2 (l.302-313).  This
module only marshals arguments.  Pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SRCS = [os.path.join(_HERE, "oracle.c"), os.path.join(_ROOT, "ptdr_inputs", "gen.c")]
_LIB = os.path.join(_HERE, "liboracle.so")

ACC_DENSE, ACC_GENERATED, ACC_DIAG, ACC_TRIDIAG, ACC_ANTIDIAG, ACC_BAND = 0, 1, 2, 3, 4, 5
LETTERS = "IXYZ"  # text-lexicographic order, code = index

_lib = None


def build(force: bool = False) -> str:
    stale = not os.path.exists(_LIB) or any(
        os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS)
    if force or stale:
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB] + _SRCS + ["-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32, u64 = ctypes.c_int, ctypes.c_uint64
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_compose.argtypes = [i32, ctypes.POINTER(ctypes.c_uint8),
                                       ctypes.POINTER(ctypes.c_uint32),
                                       ctypes.POINTER(ctypes.c_int8), ctypes.POINTER(ctypes.c_int)]
        lib.oracle_coeffs.argtypes = [i32, i32, dp, dp, dp, u64, i32,
                                      ctypes.POINTER(ctypes.c_uint64), u64, dp]
        lib.oracle_decompose.argtypes = [i32, i32, dp, dp, dp, u64, i32, dp]
        lib.oracle_frobenius2_dense.argtypes = [i32, dp]
        lib.oracle_frobenius2_dense.restype = ctypes.c_double
        lib.oracle_omp_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def threads() -> int:
    return int(_load().oracle_omp_threads())


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def string_of(q: int, n: int) -> str:
    """Text form of string index q: leftmost letter = sigma_{n-1}."""
    return "".join(LETTERS[(q >> (2 * l)) & 3] for l in reversed(range(n)))


def q_of_string(s: str) -> int:
    n = len(s)
    return sum(LETTERS.index(ch) << (2 * (n - 1 - p)) for p, ch in enumerate(s))


def compose(text: str):
    """PauliComposer: returns (k, m, n_Y) of the string `text`."""
    n = len(text)
    codes = (ctypes.c_uint8 * n)(*[LETTERS.index(c) for c in text])
    k = np.zeros(1 << n, dtype=np.uint32)
    m = np.zeros(1 << n, dtype=np.int8)
    ny = ctypes.c_int()
    rc = _load().oracle_compose(n, codes, k.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                m.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), ctypes.byref(ny))
    if rc != 0:
        raise ValueError("bad string")
    return k, m, ny.value


def _as_dense(A):
    A = np.ascontiguousarray(A, dtype=np.complex128)
    N = A.shape[0]
    n = N.bit_length() - 1
    if A.shape != (N, N) or (1 << n) != N:
        raise ValueError("A must be 2^n x 2^n")
    return A, n


def decompose(A) -> np.ndarray:
    """All 4^n coefficients of dense A in q order (complex128 [4^n])."""
    A, n = _as_dense(A)
    out = np.empty(1 << (2 * n), dtype=np.complex128)
    rc = _load().oracle_decompose(ACC_DENSE, n, _dp(A.view(np.float64)), None, None, 0, 0,
                                  _dp(out.view(np.float64)))
    if rc != 0:
        raise RuntimeError("oracle_decompose failed")
    return out


def _coeffs(kind, n, a, sub, sup, seed, variant, qs):
    qs = np.ascontiguousarray(qs, dtype=np.uint64)
    out = np.empty(qs.size, dtype=np.complex128)
    rc = _load().oracle_coeffs(kind, n, _dp(a), _dp(sub), _dp(sup), seed, variant,
                               qs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), qs.size,
                               _dp(out.view(np.float64)))
    if rc != 0:
        raise RuntimeError("oracle_coeffs failed")
    return out


def coeffs_dense(A, qs) -> np.ndarray:
    A, n = _as_dense(A)
    return _coeffs(ACC_DENSE, n, A.view(np.float64), None, None, 0, 0, qs)


def coeffs_generated(n: int, seed: int, variant: int, qs) -> np.ndarray:
    """Coefficients with entries generated on the fly by ptdr_inputs."""
    return _coeffs(ACC_GENERATED, n, None, None, None, seed, variant, qs)


def coeffs_diagonal(d, qs) -> np.ndarray:
    d = np.ascontiguousarray(d, dtype=np.complex128)
    n = d.size.bit_length() - 1
    return _coeffs(ACC_DIAG, n, d.view(np.float64), None, None, 0, 0, qs)


def coeffs_tridiagonal(sub, main, sup, qs) -> np.ndarray:
    sub, main, sup = (np.ascontiguousarray(v, dtype=np.complex128) for v in (sub, main, sup))
    n = main.size.bit_length() - 1
    return _coeffs(ACC_TRIDIAG, n, main.view(np.float64), sub.view(np.float64),
                   sup.view(np.float64), 0, 0, qs)


def coeffs_antidiagonal(a, qs) -> np.ndarray:
    """a[i] = A[i][2^n - 1 - i] (anti-diagonal storage)."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n = a.size.bit_length() - 1
    return _coeffs(ACC_ANTIDIAG, n, a.view(np.float64), None, None, 0, 0, qs)


def coeffs_band(diags, s: int, qs) -> np.ndarray:
    """(2s+1)-band storage diags[d + s][i] = A[i][i + d]."""
    diags = np.ascontiguousarray(diags, dtype=np.complex128)
    if diags.ndim != 2 or diags.shape[0] != 2 * s + 1:
        raise ValueError("diags must be [2s+1][2^n]")
    n = diags.shape[1].bit_length() - 1
    return _coeffs(ACC_BAND, n, diags.view(np.float64), None, None, 0, s, qs)


def frobenius2(A) -> float:
    A, n = _as_dense(A)
    return float(_load().oracle_frobenius2_dense(n, _dp(A.view(np.float64))))
