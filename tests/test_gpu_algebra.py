"""GPU parity of the decomposition algebra and the inverse transform (SURVEY 8(f) row f3,
PAPER.md Sec. IV-B l.521-627, and A = sum_P alpha_P P, l.116-121).

Expected values come from the oracle (the definition Tr(P A)/2^n on the composed matrix)
or from the input matrix itself (round trip); nothing is taken from the CUDA path.
"""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs
from tests.paulis import kron_string, all_strings

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _torch():
    import torch

    return torch


def _cplx(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _gpu(a):
    return _torch().from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_reconstruct_vs_kronecker(gpu, n):
    """Coefficients -> matrix on the GPU == sum_P c_P (explicit Kronecker P) for random c."""
    rng = np.random.default_rng(50 + n)
    c = _cplx(rng, 4 ** n)
    want = sum(cc * kron_string(s) for cc, s in zip(c, all_strings(n)))
    got = ptdr.reconstruct(_gpu(c)).cpu().numpy()
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(want)) * 4 ** n


@pytest.mark.parametrize("n", [1, 3, 5, 6, 8, 9, 10, 11])
def test_reconstruct_inverts_oracle(gpu, n):
    """reconstruct(oracle coefficients of A) == A (Theorem 1 uniqueness, l.98-121)."""
    A = ptdr_inputs.dense(n, 60 + n, "general")
    c = oracle.decompose(A)
    got = ptdr.reconstruct(_gpu(c)).cpu().numpy()
    assert np.max(np.abs(got - A)) <= 1e-12 * np.max(np.abs(A)) * n


@pytest.mark.parametrize("n", [12, 13, 14, 15])
def test_round_trip_large(gpu, n):
    """Full-size round trip A -> decompose -> reconstruct on the device (a property that
    holds at any size), at the bench configuration n = 15."""
    torch = _torch()
    A = ptdr.generate_dense(n, 4, "general")
    c = ptdr.decompose(A)
    B = ptdr.reconstruct(c)
    del c
    torch.cuda.empty_cache()
    err = 0.0
    for i in range(0, A.shape[0], 2048):
        err = max(err, torch.max(torch.abs(A[i:i + 2048] - B[i:i + 2048])).item())
    maxabs = max(torch.max(torch.abs(A[i:i + 2048])).item() for i in range(0, A.shape[0], 2048))
    assert err <= 1e-12 * maxabs * n, err
    del A, B
    torch.cuda.empty_cache()


def test_round_trip_n16_q_order(gpu):
    """n = 16 (64 GiB of coefficients, 64 GiB out): the q-order inverse runs in the pipeline's
    2 GiB scratch, so A -> coefficients -> A fits one GPU; compared with the generator's rows
    regenerated block by block."""
    torch = _torch()
    n, seed = 16, 5
    A = ptdr.generate_dense(n, seed, "general")
    maxabs = max(torch.max(torch.abs(A[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    c = ptdr.decompose(A)
    del A
    torch.cuda.empty_cache()
    B = ptdr.reconstruct(c)
    del c
    torch.cuda.empty_cache()
    err = 0.0
    blk = 4096
    for r0 in range(0, 1 << n, blk):
        ref = ptdr.generate_dense(n, seed, "general", row0=r0, nrows=blk)
        err = max(err, torch.max(torch.abs(B[r0:r0 + blk] - ref)).item())
        del ref
    del B
    torch.cuda.empty_cache()
    assert err <= 1e-12 * maxabs * n, err


def test_axpby_is_linear_combination(gpu):
    # l.570-577: c(mu A + nu B) = mu c(A) + nu c(B)
    rng = np.random.default_rng(71)
    n = 6
    A, B = _cplx(rng, (1 << n, 1 << n)), _cplx(rng, (1 << n, 1 << n))
    mu, nu = 0.75 - 2.0j, -1.5 + 0.25j
    got = ptdr.axpby(mu, _gpu(oracle.decompose(A)), nu, _gpu(oracle.decompose(B))).cpu().numpy()
    want = oracle.decompose(mu * A + nu * B)
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(mu * A + nu * B)) * 4


@pytest.mark.parametrize("k", [1, 2, 3])
def test_block_diag_and_direct_sum(gpu, k):
    # l.524-568: decomposition of diag(A_0..A_{2^k-1}) from those of the blocks
    rng = np.random.default_rng(80 + k)
    n = 4
    N = 1 << n
    As = [_cplx(rng, (N, N)) for _ in range(1 << k)]
    big = np.zeros((N << k, N << k), dtype=np.complex128)
    for j, Aj in enumerate(As):
        big[j * N:(j + 1) * N, j * N:(j + 1) * N] = Aj
    blocks = _gpu(np.stack([oracle.decompose(Aj) for Aj in As]))
    got = ptdr.block_diag(blocks).cpu().numpy()
    want = oracle.decompose(big)
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(big))
    if k == 1:
        ds = ptdr.direct_sum(blocks[0], blocks[1]).cpu().numpy()
        assert np.array_equal(ds, got)


def test_hermitian_augmentation(gpu):
    # l.590-627: [[0, A^*], [A, 0]] = X (x) Re(alpha) + Y (x) Im(alpha)
    rng = np.random.default_rng(90)
    n = 5
    N = 1 << n
    A = _cplx(rng, (N, N))
    aug = np.zeros((2 * N, 2 * N), dtype=np.complex128)
    aug[:N, N:] = A.conj().T
    aug[N:, :N] = A
    got = ptdr.hermitian_augment(_gpu(oracle.decompose(A))).cpu().numpy()
    want = oracle.decompose(aug)
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(A))
    assert np.all(got.imag == 0)
