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
