"""Maximum sizes of the structured paths (ptdr_max_n = 28 for band storage): the whole
decomposition on the device, checked by Parseval (Theorem 1, any size) and by oracle values
at sampled strings, with the band regenerated on the host by the independent input module
(the oracle never sees device-produced data)."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _torch():
    import torch

    return torch


def _sumsq(t):
    torch = _torch()
    flat = torch.view_as_real(t.reshape(-1))
    tot = 0.0
    for i in range(0, flat.shape[0], 1 << 27):
        c = flat[i:i + (1 << 27)]
        tot += torch.sum(c * c).item()
    return tot


@pytest.mark.parametrize("variant", ["diagonal", "tridiagonal", "anti_diagonal"])
def test_band_max_n28(gpu, variant):
    torch = _torch()
    n, seed = 28, 3
    gen_variant = "diagonal" if variant == "anti_diagonal" else variant
    band = ptdr.generate_band(n, seed, gen_variant)
    out = ptdr.decompose(band, variant)
    torch.cuda.synchronize()
    rel = abs(_sumsq(out) - _sumsq(band) / (1 << n)) / (_sumsq(band) / (1 << n))
    assert rel < 1e-11, rel
    rng = np.random.default_rng(28)
    nb = n + 1 if variant == "tridiagonal" else 1
    # 256 samples (each an O(2^28) oracle trace, ~30 s on 16 host cores) incl. every block
    blocks = np.concatenate([np.arange(nb), rng.integers(0, nb, 256 - nb)])
    zs = rng.integers(0, 1 << n, 256)
    got = out[torch.from_numpy((blocks * (1 << n) + zs).astype(np.int64)).cuda()].cpu().numpy()
    del out, band
    torch.cuda.empty_cache()
    if variant == "tridiagonal":
        xs = [(1 << int(b)) - 1 for b in blocks]
    elif variant == "diagonal":
        xs = [0] * len(blocks)
    else:
        xs = [(1 << n) - 1] * len(blocks)
    qs = np.array([ptdr.q_of(int(x), int(z), n) for x, z in zip(xs, zs)], dtype=np.uint64)
    if variant == "tridiagonal":
        sub, main, sup = ptdr_inputs.band(n, seed, "tridiagonal")
        want = oracle.coeffs_tridiagonal(sub, main, sup, qs)
        maxabs = max(np.max(np.abs(main)), np.max(np.abs(sup)))
    else:
        d = ptdr_inputs.band(n, seed, "diagonal")
        want = oracle.coeffs_diagonal(d, qs) if variant == "diagonal" else oracle.coeffs_antidiagonal(d, qs)
        maxabs = np.max(np.abs(d))
    assert np.max(np.abs(got - want)) <= TOL * maxabs


def test_band_s2_n26(gpu):
    torch = _torch()
    n, s = 26, 2
    rng = np.random.default_rng(26)
    diags = rng.standard_normal((2 * s + 1, 1 << n)) + 1j * rng.standard_normal((2 * s + 1, 1 << n))
    D = torch.from_numpy(diags).cuda()
    out = ptdr.decompose_band(D, s)
    torch.cuda.synchronize()
    # Parseval over the band matrix: sum of |stored entries| that lie inside the matrix
    N = 1 << n
    fro2 = sum(np.sum(np.abs(diags[d + s, max(0, -d):N - max(0, d)]) ** 2) for d in range(-s, s + 1))
    rel = abs(_sumsq(out) - fro2 / N) / (fro2 / N)
    assert rel < 1e-11, rel
    xs = ptdr.band_xmasks(n, s)
    b = rng.integers(0, len(xs), 24)
    z = rng.integers(0, N, 24)
    got = out[torch.from_numpy(b * N + z).cuda()].cpu().numpy()
    del out, D
    torch.cuda.empty_cache()
    qs = np.array([ptdr.q_of(int(xs[i]), int(zz), n) for i, zz in zip(b, z)], dtype=np.uint64)
    want = oracle.coeffs_band(diags, s, qs)
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(diags))
