"""In-place decomposition (ptdr_decompose_inplace_async; BASELINE.json configs[4] "n=16 ... at
1 GPU in-place"; R12): A is overwritten with its coefficients in the matrix layout
A[z][z ^ x] = alpha(x, z).  The values must be bitwise those of the out-of-place call (same
kernels, same schedule), for every kernel regime; n = 16 runs in 64 GiB + 2 GiB on one GPU
and is checked against the oracle at sampled strings plus Parseval."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def _flat_map(n):
    """q -> flat matrix-layout index, on the device."""
    torch = _torch()
    q = torch.arange(4 ** n, device="cuda", dtype=torch.int64)
    x = torch.zeros_like(q)
    z = torch.zeros_like(q)
    for l in range(n):
        c = (q >> (2 * l)) & 3
        zl = c >> 1
        x |= ((c & 1) ^ zl) << l
        z |= zl << l
    return (z << n) | (z ^ x)


@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
@pytest.mark.parametrize("n", [1, 3, 5, 6, 8, 9, 10, 11, 12, 13])
def test_inplace_bitwise_equals_out_of_place(gpu, n, variant):
    torch = _torch()
    A = ptdr.generate_dense(n, 5, variant)
    ref = ptdr.decompose(A, variant)
    B = A.clone()
    ret = ptdr.decompose(B, variant, inplace=True)
    assert ret.data_ptr() == B.data_ptr()
    got = B.reshape(-1)[_flat_map(n)]
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))
    del A, B, ref, got
    torch.cuda.empty_cache()


def test_inplace_n16_one_gpu(gpu):
    """BASELINE configs[4]: n = 16 (64 GiB) decomposed in place on one GPU."""
    torch = _torch()
    n, seed = 16, 4
    fro2 = ptdr.fro2_partials()
    A = ptdr.generate_dense(n, seed, "general", fro2=fro2)
    maxabs = max(torch.max(torch.abs(A[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    ptdr.decompose(A, "general", inplace=True)
    torch.cuda.synchronize()
    rel = abs(ptdr.sumsq(A) - ptdr.fro2_total(fro2) / (1 << n)) / (ptdr.fro2_total(fro2) / (1 << n))
    assert rel < 1e-11, rel
    rng = np.random.default_rng(1616)
    qs = np.concatenate([np.array([0, 4 ** n - 1, 1, 2, 3], dtype=np.uint64),
                         rng.integers(0, 4 ** n, 4091, dtype=np.uint64)])
    idx = ptdr.q_to_matrix_flat(qs.astype(np.int64), n)
    got = A.reshape(-1)[torch.from_numpy(idx).cuda()].cpu().numpy()
    del A
    torch.cuda.empty_cache()
    want = oracle.coeffs_generated(n, seed, ptdr_inputs.VARIANTS["general"], qs)
    assert np.max(np.abs(got - want)) <= 1e-12 * maxabs


def test_inplace_rejects_band_structures(gpu):
    torch = _torch()
    d = torch.zeros(1 << 6, dtype=torch.complex128, device="cuda")
    with pytest.raises(ptdr.PtdrError):
        ptdr.decompose(d, "diagonal", inplace=True)


@pytest.mark.parametrize("variant", ["general", "hermitian"])
@pytest.mark.parametrize("n", [4, 9, 12, 14])
def test_matrix_layout_out_of_place(gpu, n, variant):
    """ptdr_decompose_matrix_layout_async: the in-place layout written to a separate buffer,
    bitwise the permuted q-order result; A untouched."""
    torch = _torch()
    A = ptdr.generate_dense(n, 6, variant)
    keep = A.clone()
    ref = ptdr.decompose(A, variant)
    M = ptdr.decompose_matrix_layout(A, variant)
    assert torch.equal(torch.view_as_real(A), torch.view_as_real(keep))
    assert torch.equal(torch.view_as_real(M.reshape(-1)[_flat_map(n)]), torch.view_as_real(ref))
