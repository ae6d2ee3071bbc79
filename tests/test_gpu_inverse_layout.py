"""GPU parity of the inverse transform from the matrix layout (ptdr_reconstruct_matrix_layout_async;
A = sum_P alpha_P P).  The input is the layout the in-place decomposition
writes, M[z][z ^ x] = alpha(x, z); n >= 11 runs the forward TMA pipeline with the phase
(-i)^{popcount(x & z)} applied on input, smaller n the q-order inverse.

Expected values come from the explicit Kronecker sum, from the input matrix of an oracle
decomposition, or from the input matrix itself (round trip); nothing is taken from the CUDA
path."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs
from tests.paulis import kron_string, all_strings

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def _to_layout(c, n):
    """q-ordered coefficients -> matrix layout M[z][z ^ x] (host index map of the binding)."""
    M = np.empty(4 ** n, dtype=np.complex128)
    M[ptdr.q_to_matrix_flat(np.arange(4 ** n, dtype=np.int64), n)] = c
    return M.reshape(1 << n, 1 << n)


def _gpu(a):
    return _torch().from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_vs_kronecker(gpu, n):
    rng = np.random.default_rng(70 + n)
    c = rng.standard_normal(4 ** n) + 1j * rng.standard_normal(4 ** n)
    want = sum(cc * kron_string(s) for cc, s in zip(c, all_strings(n)))
    got = ptdr.reconstruct_matrix_layout(_gpu(_to_layout(c, n))).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want)) * 4 ** n


@pytest.mark.parametrize("n", [1, 3, 5, 6, 8, 9, 10, 11, 12])
def test_inverts_oracle(gpu, n):
    """reconstruct_matrix_layout(oracle coefficients of A in the matrix layout) == A, on both
    sides of the pipeline threshold (n = 11, 12 run MODE_INV)."""
    A = ptdr_inputs.dense(n, 80 + n, "general")
    M = _to_layout(oracle.decompose(A), n)
    got = ptdr.reconstruct_matrix_layout(_gpu(M)).cpu().numpy()
    assert np.max(np.abs(got - A)) <= 1e-12 * np.max(np.abs(A)) * n


@pytest.mark.parametrize("variant", ["general", "hermitian"])
@pytest.mark.parametrize("n", [6, 11, 12, 13, 14, 15])
def test_round_trip_and_in_place(gpu, n, variant):
    """A -> decompose_matrix_layout -> reconstruct_matrix_layout == A (any size), and the
    in-place call is bitwise the out-of-place one."""
    torch = _torch()
    A = ptdr.generate_dense(n, 9, variant)
    M = ptdr.decompose_matrix_layout(A, variant)
    B = ptdr.reconstruct_matrix_layout(M)
    err = 0.0
    maxabs = 0.0
    for i in range(0, A.shape[0], 2048):
        err = max(err, torch.max(torch.abs(A[i:i + 2048] - B[i:i + 2048])).item())
        maxabs = max(maxabs, torch.max(torch.abs(A[i:i + 2048])).item())
    assert err <= 1e-12 * maxabs * n, err
    del A
    ret = ptdr.reconstruct_matrix_layout(M, inplace=True)
    assert ret.data_ptr() == M.data_ptr()
    assert torch.equal(torch.view_as_real(M), torch.view_as_real(B))
    del M, B
    torch.cuda.empty_cache()


def test_in_place_round_trip_n16(gpu):
    """BASELINE configs[4]'s one-GPU in-place size: A (64 GiB) -> coefficients -> A, in place
    both ways, against a second copy generated from the same seed."""
    torch = _torch()
    n, seed = 16, 3
    A = ptdr.generate_dense(n, seed, "general")
    ptdr.decompose(A, "general", inplace=True)
    ptdr.reconstruct_matrix_layout(A, inplace=True)
    ref = ptdr.generate_dense(n, seed, "general")
    err = 0.0
    maxabs = 0.0
    for i in range(0, ref.shape[0], 1024):
        err = max(err, torch.max(torch.abs(A[i:i + 1024] - ref[i:i + 1024])).item())
        maxabs = max(maxabs, torch.max(torch.abs(ref[i:i + 1024])).item())
    del A, ref
    torch.cuda.empty_cache()
    assert err <= 1e-12 * maxabs * n, err


def test_errors(gpu):
    torch = _torch()
    M = torch.zeros((1 << 12, 1 << 12), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        ptdr.reconstruct_matrix_layout(M, out=M, inplace=True)
    flat = torch.zeros(2 * 4 ** 12, dtype=torch.complex128, device="cuda")
    with pytest.raises(ptdr.PtdrError):   # partial overlap of M and A
        ptdr.reconstruct_matrix_layout(flat[:4 ** 12], out=flat[4 ** 11:4 ** 11 + 4 ** 12])
