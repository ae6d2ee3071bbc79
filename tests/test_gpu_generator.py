"""GPU generator kernel (row a1) vs the host input module (independent code).

Philox integers are identical by construction; the Box-Muller floats may differ
by a few ulp (CUDA vs glibc log/sincos), so the check is |d| <= 8 ulp-ish."""
import numpy as np
import pytest

import paper_2403_11644_b200 as ptdr
import ptdr_inputs

pytestmark = pytest.mark.gpu


def _close(a, b):
    return np.max(np.abs(a - b)) <= 4e-15 * max(1.0, np.max(np.abs(b)))


@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_dense_generator_matches_host(gpu, variant):
    n = 9
    got = ptdr.generate_dense(n, 4, variant).cpu().numpy()
    want = ptdr_inputs.dense(n, 4, variant)
    assert _close(got, want)
    if variant == "hermitian":
        assert np.array_equal(got, got.conj().T)       # exact on the device too
    part = ptdr.generate_dense(n, 4, variant, row0=100, nrows=7).cpu().numpy()
    assert np.array_equal(part, got[100:107])          # row split does not change values


def test_band_generator_matches_host(gpu):
    n = 12
    got = ptdr.generate_band(n, 3, "tridiagonal").cpu().numpy()
    sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
    assert _close(got, np.stack([sub, main, sup]))
    d = ptdr.generate_band(n, 3, "diagonal").cpu().numpy()
    assert _close(d, ptdr_inputs.band(n, 3, "diagonal"))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sendblocks_layout(gpu, world):
    n = 8
    N, R = 1 << n, (1 << n) // world
    A = ptdr.generate_dense(n, 4, "general").cpu().numpy()
    for rank in range(world):
        s = ptdr.generate_sendblocks(n, 4, rank, world).cpu().numpy().reshape(world, R, R)
        for b in range(world):
            want = A[rank * R:(rank + 1) * R, (rank ^ b) * R:((rank ^ b) + 1) * R]
            assert np.array_equal(s[b], want)


@pytest.mark.parametrize("world,K", [(2, 2), (2, 4), (4, 2), (8, 4), (1, 4)])
def test_sendblocks_subrange_layout(gpu, world, K):
    """[K][world][K][R'][R'] layout: element (s, h, t, r', c') =
    A[(rank K + t) R' + r'][((rank ^ h) K + (t ^ s)) R' + c'] (include/ptdr.h)."""
    n = 9
    N, R = 1 << n, (1 << n) // world
    Rp = R // K
    A = ptdr.generate_dense(n, 4, "general").cpu().numpy()
    for rank in range(world):
        s = ptdr.generate_sendblocks(n, 4, rank, world, subranges=K).cpu().numpy()
        s = s.reshape(K, world, K, Rp, Rp)
        for sr in range(K):
            for h in range(world):
                for t in range(K):
                    r0 = (rank * K + t) * Rp
                    c0 = ((rank ^ h) * K + (t ^ sr)) * Rp
                    assert np.array_equal(s[sr, h, t], A[r0:r0 + Rp, c0:c0 + Rp])


@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_generator_fro2_partials(gpu, variant):
    """The fused ||A||_F^2 partials equal a sum over the written matrix (and a row block)."""
    import torch

    n = 11
    f = ptdr.fro2_partials()
    A = ptdr.generate_dense(n, 4, variant, fro2=f)
    want = float(torch.sum(torch.abs(A) ** 2).item())
    assert abs(ptdr.fro2_total(f) - want) <= 1e-12 * want
    assert abs(ptdr.sumsq(A) - want) <= 1e-12 * want
    part = ptdr.generate_dense(n, 4, variant, row0=64, nrows=100, fro2=f)
    want = float(torch.sum(torch.abs(part) ** 2).item())
    assert abs(ptdr.fro2_total(f) - want) <= 1e-12 * want
    B = ptdr.generate_band(12, 3, "tridiagonal", fro2=f)
    want = float(torch.sum(torch.abs(B) ** 2).item())
    assert abs(ptdr.fro2_total(f) - want) <= 1e-12 * want
    S = ptdr.generate_sendblocks(10, 4, 1, 4, subranges=2, fro2=f)
    want = float(torch.sum(torch.abs(S) ** 2).item())
    assert abs(ptdr.fro2_total(f) - want) <= 1e-12 * want
