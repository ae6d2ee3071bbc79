"""The HERMITIAN / REAL_SYMMETRIC contract (include/ptdr.h; R9): only the upper
triangle is read -- plus the real part of the diagonal (HERMITIAN), or only real parts
(REAL_SYMMETRIC).  Every element the contract says is not read is overwritten with NaN;
the result must be bit-identical to the clean input's (a single NaN read anywhere would
propagate into a coefficient).  Sizes cover every kernel regime: the direct kernel
(n <= 5), whole-vector tiles (n = 6..10) incl. the mirrored launch, and the TMA pipeline's
half-length modes (n >= 11)."""
import numpy as np
import pytest

import paper_2403_11644_b200 as ptdr

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


def _poison(A, variant):
    torch = _torch()
    P = A.clone()
    N = A.shape[0]
    Pr = torch.view_as_real(P)                      # [N][N][2]
    lower = torch.tril(torch.ones(N, N, dtype=torch.bool, device=A.device), -1)
    Pr[lower] = float("nan")                        # strict lower triangle: re and im
    idx = torch.arange(N, device=A.device)
    Pr[idx, idx, 1] = float("nan")                  # Im of the diagonal
    if variant == "real_symmetric":
        Pr[..., 1] = float("nan")                   # every imaginary part
    return P


@pytest.mark.parametrize("variant", ["hermitian", "real_symmetric"])
@pytest.mark.parametrize("n", [1, 3, 5, 6, 8, 9, 10, 11, 12, 13])
def test_unread_triangle_is_never_read(gpu, n, variant):
    torch = _torch()
    A = ptdr.generate_dense(n, 2, variant)
    clean = ptdr.decompose(A, variant)
    dirty = ptdr.decompose(_poison(A, variant), variant)
    torch.cuda.synchronize()
    assert not torch.isnan(torch.view_as_real(dirty)).any()
    assert torch.equal(torch.view_as_real(clean), torch.view_as_real(dirty))
    assert torch.all(dirty.imag == 0)
    del A, clean, dirty
    torch.cuda.empty_cache()


def test_unread_triangle_n15(gpu):
    """The largest Hermitian bench size (n = 15, 16 GiB): poison in place in row blocks."""
    torch = _torch()
    n, variant = 15, "hermitian"
    A = ptdr.generate_dense(n, 4, variant)
    clean = ptdr.decompose(A, variant)
    N = A.shape[0]
    Ar = torch.view_as_real(A)
    for r0 in range(0, N, 2048):
        rows = torch.arange(r0, r0 + 2048, device=A.device)[:, None]
        cols = torch.arange(N, device=A.device)[None, :]
        blk = Ar[r0:r0 + 2048]
        blk[(cols < rows)] = float("nan")
        d = torch.arange(r0, r0 + 2048, device=A.device)
        Ar[d, d, 1] = float("nan")
    dirty = ptdr.decompose(A, variant)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(clean), torch.view_as_real(dirty))
    del A, clean, dirty
    torch.cuda.empty_cache()
