"""CPU checks of the C-ABI library: it loads and exports every declared symbol,
and its pure host functions (sizes, workspace, validation) behave as documented.
No compute call is made here (no GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2403_11644_b200 as ptdr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    """Every function declared in include/*.h (ptdr.h and ptdr_debug.h)."""
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if not h.endswith(".h"):
            continue
        with open(os.path.join(ROOT, "include", h)) as f:
            src = f.read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(ptdr_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def L():
    from paper_2403_11644_b200 import build

    build.build()
    return ptdr.lib()


def test_exports_every_declared_symbol(L):
    syms = _declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s


def test_counts(L):
    assert ptdr.input_count(15) == 1 << 30
    assert ptdr.output_count(15) == 1 << 30
    assert ptdr.input_count(24, "diagonal") == 1 << 24
    assert ptdr.input_count(24, "tridiagonal") == 3 << 24
    assert ptdr.output_count(24, "tridiagonal") == 25 << 24
    # HERMITIAN_TRIDIAGONAL: [main, sup] in, the same n + 1 blocks out, half the segment storage
    assert ptdr.input_count(24, "hermitian_tridiagonal") == 2 << 24
    assert ptdr.output_count(24, "hermitian_tridiagonal") == 25 << 24
    assert ptdr.workspace_bytes(24, "hermitian_tridiagonal") == (1 << 24) * 16 + 256
    assert ptdr.n_of(np.zeros((2, 1 << 5), dtype=np.complex128), "hermitian_tridiagonal") == 5
    with pytest.raises(ValueError):
        ptdr.n_of(np.zeros((3, 1 << 5), dtype=np.complex128), "hermitian_tridiagonal")
    assert ptdr.output_count(0) == 0 and ptdr.output_count(17) == 0
    assert L.ptdr_max_n(0) == 16 and L.ptdr_max_n(4) == 28


def test_workspace_is_deterministic_and_small(L):
    for n in range(1, 17):
        for s in ("general", "hermitian", "real_symmetric"):
            a = ptdr.workspace_bytes(n, s)
            assert a == ptdr.workspace_bytes(n, s)
            # scratch slots are capped by a 2 GiB budget, never more
            # than the input itself
            assert a <= (2 << 30) + (1 << 20), (n, s, a)
            assert a <= 16 * 4 ** n + (1 << 20), (n, s, a)
    # band paths: 256 B of tail-pipeline counters (+ the P/M segments for the tridiagonal)
    assert ptdr.workspace_bytes(24, "diagonal") == 256
    assert ptdr.workspace_bytes(24, "tridiagonal") == 2 * (1 << 24) * 16 + 256
    with pytest.raises(ptdr.PtdrError):
        ptdr.workspace_bytes(15, "hermitian", 2)     # sharding is GENERAL only
    with pytest.raises(ptdr.PtdrError):
        ptdr.workspace_bytes(15, "general", 3)       # world must be a power of two
    assert ptdr.workspace_bytes(15, "general", 8) > 0


def test_validation_without_gpu(L):
    # argument validation happens before any CUDA call
    st = L.ptdr_decompose_async(None, 5, 0, None, None, 0, None)
    assert st == ptdr.PTDR_EINVAL
    st = L.ptdr_decompose_async(ctypes.c_void_p(16), 0, 0, ctypes.c_void_p(4096), None, 0, None)
    assert st == ptdr.PTDR_EINVAL                   # n = 0 rejected
    st = L.ptdr_decompose_async(ctypes.c_void_p(8), 3, 0, ctypes.c_void_p(4096), None, 0, None)
    assert st == ptdr.PTDR_EINVAL                   # misaligned
    st = L.ptdr_decompose_async(ctypes.c_void_p(4096), 3, 0, ctypes.c_void_p(4096 + 64), None, 0,
                                None)
    assert st == ptdr.PTDR_EUNSUPPORTED             # out overlaps A
    st = L.ptdr_decompose_async(ctypes.c_void_p(1 << 20), 12, 0, ctypes.c_void_p(1 << 30), None, 0,
                                None)
    assert st == ptdr.PTDR_ENOMEM                   # workspace required
    assert b"workspace" in L.ptdr_last_error()
    st = L.ptdr_decompose_xshard_async(ctypes.c_void_p(4096), 10, 0, 3, ctypes.c_void_p(1 << 30),
                                       None, 0, None)
    assert st == ptdr.PTDR_EINVAL
    assert L.ptdr_status_string(3) == b"PTDR_ENOMEM"


def test_q_helpers_roundtrip():
    import oracle

    n = 4
    for q in range(4 ** n):
        x, z = ptdr.xz_of(q, n)
        assert ptdr.q_of(x, z, n) == q
        s = oracle.string_of(q, n)
        # X-mask bit l set iff sigma_l in {X,Y}; Z-mask bit l set iff sigma_l in {Y,Z}
        for l in range(n):
            ch = s[n - 1 - l]
            assert ((x >> l) & 1) == (ch in "XY")
            assert ((z >> l) & 1) == (ch in "YZ")


def test_plan_validation_without_gpu(L):
    """ptdr_plan_create validates its arguments before touching the device."""
    h = ctypes.c_void_p()
    assert L.ptdr_plan_create(0, 0, 2, ctypes.byref(h)) == ptdr.PTDR_EINVAL      # n = 0
    assert L.ptdr_plan_create(17, 0, 2, ctypes.byref(h)) == ptdr.PTDR_EINVAL     # n > 16 dense
    assert L.ptdr_plan_create(10, 0, 0, ctypes.byref(h)) == ptdr.PTDR_EINVAL     # depth 0
    assert L.ptdr_plan_create(10, 0, 5, ctypes.byref(h)) == ptdr.PTDR_EINVAL     # depth > 4
    assert L.ptdr_plan_create(10, 9, 1, ctypes.byref(h)) == ptdr.PTDR_EINVAL     # structure
    assert L.ptdr_plan_create(10, 0, 1, None) == ptdr.PTDR_EINVAL                # null out
    assert L.ptdr_plan_wait(None) == ptdr.PTDR_EINVAL
    assert L.ptdr_plan_destroy(None) == ptdr.PTDR_OK


@pytest.mark.parametrize("s", [0, 1, 2, 3, 4, 5, 8])
def test_band_xmask_list_matches_definition(L, s):
    """Host planner of BAND(s): the block list is {0} U {i ^ (i+d) : 1 <= d <= s}, ascending,
    of size s n - c(s) (PAPER Table I, l.500-518) -- brute force for small n, count for large."""
    import numpy as np

    for n in range(max(1, s.bit_length()), 11):
        if (1 << n) <= s:
            continue
        xs = ptdr.band_xmasks(n, s)
        N = 1 << n
        want = sorted({0} | {i ^ (i + d) for d in range(1, s + 1) for i in range(N - d)})
        assert xs.tolist() == want, (n, s)
    if s >= 1:
        Lg = s.bit_length() - 1
        cs = s * (Lg + 1) - (1 << (Lg + 1))
        for n in (16, 24, 28):
            assert L.ptdr_band_xmask_count(n, s) == s * n - cs
    assert L.ptdr_band_xmask_count(0, s) == 0
    assert L.ptdr_band_xmask_count(29, s) == 0


def test_anti_diagonal_counts(L):
    assert ptdr.input_count(10, "anti_diagonal") == 1 << 10
    assert ptdr.output_count(10, "anti_diagonal") == 1 << 10
    assert ptdr.workspace_bytes(24, "anti_diagonal") == 256
    assert L.ptdr_max_n(5) == 28


def test_padded_workspace_rules(L):
    """Zero padding: m = 0 is invalid; powers of two need no pad buffer;
    GENERAL at n >= 11 reads in place; everything else adds a 2^n x 2^n pad buffer."""
    inval = ctypes.c_size_t(-1).value
    assert L.ptdr_padded_workspace_bytes(0, 0) == inval
    assert L.ptdr_padded_workspace_bytes(65537, 0) == inval
    assert L.ptdr_padded_workspace_bytes(5, 3) == inval                        # band structure
    # exact powers of two cover the zero-padded copy too (a strided view, lda != m, takes it)
    assert L.ptdr_padded_workspace_bytes(1024, 0) >= 16 * 4 ** 10 + ptdr.workspace_bytes(10, "general")
    assert L.ptdr_padded_workspace_bytes(1024, 1) >= 16 * 4 ** 10 + ptdr.workspace_bytes(10, "hermitian")
    assert L.ptdr_padded_workspace_bytes(16, 0) >= 16 * 4 ** 4
    assert L.ptdr_padded_workspace_bytes(32768, 1) >= 16 * 4 ** 15
    # GENERAL on the TMA pipeline reads any pitch in place: no copy
    assert L.ptdr_padded_workspace_bytes(4096, 0) == ptdr.workspace_bytes(12, "general")
    assert L.ptdr_padded_workspace_bytes(3000, 0) == ptdr.workspace_bytes(12, "general")
    assert L.ptdr_padded_workspace_bytes(1000, 0) >= 16 * 4 ** 10
    assert L.ptdr_padded_workspace_bytes(3000, 1) >= 16 * 4 ** 12 + ptdr.workspace_bytes(12, "hermitian")


def test_structure_enum_matches_binding():
    """The binding's structure names map to the values include/ptdr.h declares."""
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ptdr.h")).read()
    enum = dict((name.lower(), int(v)) for name, v in re.findall(r"PTDR_([A-Z_]+)\s*=\s*(\d+)", hdr.split("} ptdr_structure;")[0].split("typedef enum {")[-1]))
    assert enum == ptdr.STRUCTURES
