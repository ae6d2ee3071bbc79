"""Seeded synthetic input generator (host side) -- shared by tests, oracle and bench.

Holds none of the decomposition arithmetic: it only produces the matrices the
paper's experiments use ("a generic matrix, with no specific structure",
PAPER.md l.631; entries "from a function", l.646).  The recipe (Philox4x32-10 +
Box-Muller, one counter per global element index) is documented in gen.c and
in DESIGN.md "Input recipe".  The CUDA generator kernel is an independent
implementation of the same recipe (checked against this module in
tests/test_gpu_generator.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libptdr_inputs.so")

GENERAL, HERMITIAN, REAL_SYMMETRIC, DIAGONAL, TRIDIAGONAL = 0, 1, 2, 3, 4
VARIANTS = {
    "general": GENERAL,
    "hermitian": HERMITIAN,
    "real_symmetric": REAL_SYMMETRIC,
    "diagonal": DIAGONAL,
    "tridiagonal": TRIDIAGONAL,
}

# Seeds per BASELINE.json configs.
CONFIG_SEEDS = {"n6": 0, "n10": 1, "n13": 2, "n24": 3, "n15": 4, "n16": 4}

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        )
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u64, i32, dp = ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)
        lib.ptdr_inputs_philox4x32_10.argtypes = [
            ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
            ctypes.POINTER(ctypes.c_uint32)]
        lib.ptdr_inputs_normal_pair.argtypes = [u64, u64, ctypes.c_uint32, dp, dp]
        lib.ptdr_inputs_entry.argtypes = [i32, u64, i32, u64, u64, dp, dp]
        lib.ptdr_inputs_dense_rows.argtypes = [i32, u64, i32, u64, u64, dp]
        lib.ptdr_inputs_band.argtypes = [i32, u64, i32, dp, dp, dp]
        _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def philox4x32_10(ctr, key) -> tuple:
    lib = _load()
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib.ptdr_inputs_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def normal_pair(seed: int, idx: int, stream: int = 0) -> complex:
    lib = _load()
    re, im = ctypes.c_double(), ctypes.c_double()
    lib.ptdr_inputs_normal_pair(seed, idx, stream, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def entry(n: int, seed: int, variant: int, row: int, col: int) -> complex:
    lib = _load()
    re, im = ctypes.c_double(), ctypes.c_double()
    lib.ptdr_inputs_entry(n, seed, variant, row, col, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def dense(n: int, seed: int, variant=GENERAL, row0: int = 0, nrows: int | None = None,
          out: np.ndarray | None = None) -> np.ndarray:
    """Rows [row0, row0+nrows) of the 2^n x 2^n matrix, complex128, row-major."""
    variant = VARIANTS.get(variant, variant)
    if variant not in (GENERAL, HERMITIAN, REAL_SYMMETRIC):
        raise ValueError("dense() takes a dense variant; use band() for diagonal/tridiagonal")
    N = 1 << n
    nrows = N - row0 if nrows is None else nrows
    if out is None:
        out = np.empty((nrows, N), dtype=np.complex128)
    assert out.dtype == np.complex128 and out.flags.c_contiguous and out.size == nrows * N
    _load().ptdr_inputs_dense_rows(n, seed, variant, row0, nrows, _dp(out.view(np.float64)))
    return out


def band(n: int, seed: int, variant=TRIDIAGONAL):
    """Band storage: DIAGONAL -> main[2^n]; TRIDIAGONAL -> (sub, main, sup), each [2^n]
    complex128, sub[i] = A[i][i-1], main[i] = A[i][i], sup[i] = A[i][i+1]."""
    variant = VARIANTS.get(variant, variant)
    N = 1 << n
    main = np.zeros(N, dtype=np.complex128)
    sub = np.zeros(N, dtype=np.complex128)
    sup = np.zeros(N, dtype=np.complex128)
    _load().ptdr_inputs_band(n, seed, variant, _dp(sub.view(np.float64)),
                             _dp(main.view(np.float64)), _dp(sup.view(np.float64)))
    if variant == DIAGONAL:
        return main
    if variant == TRIDIAGONAL:
        return sub, main, sup
    raise ValueError("band() takes diagonal or tridiagonal")


def densify_band(n: int, main, sub=None, sup=None) -> np.ndarray:
    """Dense matrix from band arrays (test helper; plain placement, no arithmetic)."""
    N = 1 << n
    A = np.zeros((N, N), dtype=np.complex128)
    idx = np.arange(N)
    A[idx, idx] = main
    if sup is not None:
        A[idx[:-1], idx[:-1] + 1] = sup[:-1]
    if sub is not None:
        A[idx[1:], idx[1:] - 1] = sub[1:]
    return A
