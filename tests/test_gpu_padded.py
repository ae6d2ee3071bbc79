"""Zero padding: an m x m matrix, m not a power of two, decomposed as the
top-left block of the 2^n x 2^n zero matrix -- the ragged sizes of the dense path.  The
expected values are the oracle's coefficients of the explicitly padded matrix."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _torch():
    import torch

    return torch


def _matrix(rng, m, variant):
    B = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    if variant == "hermitian":
        return (B + B.conj().T) / 2
    if variant == "real_symmetric":
        U = np.triu(B.real)
        return (U + np.triu(U, 1).T).astype(np.complex128)
    return B


def _padded(A):
    m = A.shape[0]
    n = max(1, (m - 1).bit_length())
    P = np.zeros((1 << n, 1 << n), dtype=np.complex128)
    P[:m, :m] = A
    return P, n


@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
@pytest.mark.parametrize("m", [1, 2, 3, 5, 7, 33, 100, 255, 600])
def test_padded_full_oracle(gpu, m, variant):
    torch = _torch()
    rng = np.random.default_rng(m * 7 + len(variant))
    A = _matrix(rng, m, variant)
    got = ptdr.decompose_padded(torch.from_numpy(A).cuda(), variant).cpu().numpy()
    P, n = _padded(A)
    want = oracle.decompose(P)
    assert got.size == 4 ** n
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(A))


@pytest.mark.parametrize("m,variant", [(1500, "general"), (3000, "general"), (2500, "hermitian"),
                                       (5000, "general")])
def test_padded_large_sampled(gpu, m, variant):
    """n = 11..13: GENERAL reads the stored block in place through TMA zero fill."""
    torch = _torch()
    rng = np.random.default_rng(m)
    A = _matrix(rng, m, variant)
    got = ptdr.decompose_padded(torch.from_numpy(A).cuda(), variant).cpu().numpy()
    P, n = _padded(A)
    qs = np.unique(np.concatenate([rng.integers(0, 4 ** n, 700), [0, 4 ** n - 1]])).astype(np.uint64)
    want = oracle.coeffs_dense(P, qs)
    assert np.max(np.abs(got[qs.astype(np.int64)] - want)) <= TOL * np.max(np.abs(A))
    # Parseval over the padded matrix (Theorem 1)
    lhs = np.sum(np.abs(got) ** 2)
    rhs = np.sum(np.abs(A) ** 2) / (1 << n)
    assert abs(lhs - rhs) / rhs < 1e-11


def test_padded_strided_view_and_power_of_two(gpu):
    """A sub-block view with row pitch > m, and an exact power of two (no padding)."""
    torch = _torch()
    rng = np.random.default_rng(5)
    big = rng.standard_normal((2100, 2100)) + 1j * rng.standard_normal((2100, 2100))
    Bt = torch.from_numpy(big).cuda()
    view = Bt[:2000, :2000]                      # m = 2000, lda = 2100, n = 11 (in place)
    got = ptdr.decompose_padded(view).cpu().numpy()
    P, n = _padded(big[:2000, :2000])
    qs = rng.integers(0, 4 ** n, 500).astype(np.uint64)
    assert np.max(np.abs(got[qs.astype(np.int64)] - oracle.coeffs_dense(P, qs))) <= TOL * np.max(np.abs(big))
    exact = Bt[:1024, :1024].contiguous()
    a = ptdr.decompose_padded(exact).cpu().numpy()
    b = ptdr.decompose(exact).cpu().numpy()
    assert np.array_equal(a, b)
    small_view = Bt[:300, :300]                  # copy path with a strided source
    got = ptdr.decompose_padded(small_view).cpu().numpy()
    P, n = _padded(big[:300, :300])
    assert np.max(np.abs(got - oracle.decompose(P))) <= TOL * np.max(np.abs(big))


def test_padded_empty_is_rejected(gpu):
    torch = _torch()
    A = torch.zeros((0, 0), dtype=torch.complex128, device="cuda")
    with pytest.raises(ptdr.PtdrError) as e:
        ptdr.decompose_padded(A)
    assert e.value.status == ptdr.PTDR_EINVAL


@pytest.mark.parametrize("m,variant", [(1024, "hermitian"), (1024, "real_symmetric"), (512, "general"),
                                       (16, "general"), (16, "hermitian")])
def test_padded_exact_size_strided_view(gpu, m, variant):
    """m = 2^n stored with row pitch > m takes the zero-padded copy: the
    workspace the size function reports must cover that copy, and the result must equal the
    contiguous decomposition bit for bit."""
    torch = _torch()
    rng = np.random.default_rng(m + len(variant))
    big = _matrix(rng, 2100, variant)
    Bt = torch.from_numpy(big).cuda()
    view = Bt[:m, :m]
    nb = int(ptdr.lib().ptdr_padded_workspace_bytes(m, ptdr.STRUCTURES[variant]))
    assert nb >= 16 * m * m
    got = ptdr.decompose_padded(view, variant).cpu().numpy()
    want = ptdr.decompose(view.contiguous(), variant).cpu().numpy()
    assert np.array_equal(got, want)
    # an exact-size workspace passes, a byte short is refused before any launch
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    got2 = ptdr.decompose_padded(view, variant, workspace=ws).cpu().numpy()
    assert np.array_equal(got2, want)
    with pytest.raises(ptdr.PtdrError) as e:
        ptdr.decompose_padded(view, variant, workspace=ws[: nb - 256])
    assert e.value.status == ptdr.PTDR_ENOMEM
