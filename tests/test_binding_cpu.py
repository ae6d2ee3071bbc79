"""CPU checks of the Python binding: argument marshalling only, and no CPU fallback --
a CPU tensor is rejected, and a missing library raises instead of computing anything."""
import importlib

import numpy as np
import pytest
import torch

import paper_2403_11644_b200 as ptdr


def test_cpu_tensors_are_rejected():
    A = torch.zeros((8, 8), dtype=torch.complex128)
    with pytest.raises(TypeError):
        ptdr.decompose(A)
    with pytest.raises(TypeError):
        ptdr.decompose_padded(A[:5, :5])
    with pytest.raises(TypeError):
        ptdr.reconstruct(torch.zeros(64, dtype=torch.complex128))
    with pytest.raises(TypeError):
        ptdr.decompose_batched(torch.zeros((2, 8, 8), dtype=torch.complex128))


def test_shape_and_dtype_validation():
    with pytest.raises(ValueError):
        ptdr.n_of(torch.zeros((6, 6)), "general")           # not a power of two
    with pytest.raises(ValueError):
        ptdr.n_of(torch.zeros((4, 8)), "general")           # not square
    assert ptdr.n_of(torch.zeros(3 << 5), "tridiagonal") == 5
    assert ptdr.n_of(torch.zeros(1 << 7), "anti_diagonal") == 7


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import paper_2403_11644_b200 as mod

    monkeypatch.setattr(mod, "_lib", None)
    monkeypatch.setattr(mod, "LIB_PATH", str(tmp_path / "libptdr_missing.so"))
    with pytest.raises(ImportError):
        mod.lib()


def test_q_order_helpers_roundtrip():
    n = 5
    for q in range(4 ** n):
        x, z = ptdr.xz_of(q, n)
        assert ptdr.q_of(x, z, n) == q


def test_band_shapes_are_validated():
    with pytest.raises(ValueError):
        ptdr.n_of(torch.zeros(3 * 5), "tridiagonal")        # 5 is not a power of two
    with pytest.raises(ValueError):
        ptdr.n_of(torch.zeros((4, 8)), "tridiagonal")       # [3, 2^n] only
    with pytest.raises(ValueError):
        ptdr.n_of(torch.zeros((2, 8)), "diagonal")          # 1-D band
    with pytest.raises(ValueError):
        ptdr.n_of(torch.zeros(0), "diagonal")


def test_host_entry_validates_sizes_before_the_abi_call():
    """decompose_host checks every size against n before passing raw host pointers (the
    ABI cannot): a non-square, non-power-of-two or wrongly sized out_host is refused."""
    with pytest.raises(ValueError):
        ptdr.decompose_host(np.zeros((4, 8), dtype=np.complex128))
    with pytest.raises(ValueError):
        ptdr.decompose_host(np.zeros((6, 6), dtype=np.complex128))
    with pytest.raises(ValueError):
        ptdr.decompose_host(np.zeros((4, 4), dtype=np.complex128), out_host=np.zeros(15, dtype=np.complex128))
    with pytest.raises(ValueError):
        ptdr.decompose_host(np.zeros(3 * 8 + 1, dtype=np.complex128), "tridiagonal")
    with pytest.raises(TypeError):
        ptdr.decompose_host(np.zeros((4, 4), dtype=np.complex64))


def test_matrix_layout_index_is_a_permutation():
    """The in-place layout puts alpha(x, z) at A[z][z ^ x]: a bijection of the 4^n slots,
    and the flat map agrees with matrix_index."""
    for n in (1, 3, 5):
        flat = ptdr.q_to_matrix_flat(np.arange(4 ** n), n)
        assert sorted(flat.tolist()) == list(range(4 ** n))
        for q in range(0, 4 ** n, 7):
            x, z = ptdr.xz_of(q, n)
            r, c = ptdr.matrix_index(x, z, n)
            assert flat[q] == r * (1 << n) + c and (r ^ c) == x
