"""GPU parity of the ANTI_DIAGONAL and BAND(s) paths vs the CPU oracle.

Inputs: seeded numpy draws (iid N(0,1) real and imaginary parts, the recipe of the other
band configurations).  Expected values come only from oracle.coeffs_antidiagonal /
oracle.coeffs_band (the definition Tr(P A)/2^n with band accessors).
"""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
from paper_2403_11644_b200 import q_of

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _torch():
    import torch

    return torch


def _cplx(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _qs_block(x, n, zs):
    return np.array([q_of(int(x), int(z), n) for z in zs], dtype=np.uint64)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 13])
def test_antidiagonal_full(gpu, n):
    torch = _torch()
    rng = np.random.default_rng(1000 + n)
    a = _cplx(rng, 1 << n)
    out = ptdr.decompose(torch.from_numpy(a).cuda(), "anti_diagonal").cpu().numpy()
    zs = np.arange(1 << n)
    want = oracle.coeffs_antidiagonal(a, _qs_block((1 << n) - 1, n, zs))
    err = np.max(np.abs(out - want))
    assert err <= TOL * np.max(np.abs(a)), err


def test_antidiagonal_n24_sampled_and_zshard(gpu):
    torch = _torch()
    n = 24
    rng = np.random.default_rng(1024)
    a = _cplx(rng, 1 << n)
    A = torch.from_numpy(a).cuda()
    out = ptdr.decompose(A, "anti_diagonal")
    zs = np.unique(np.concatenate([[0, (1 << n) - 1], rng.integers(0, 1 << n, 1000)]))
    want = oracle.coeffs_antidiagonal(a, _qs_block((1 << n) - 1, n, zs))
    got = out[torch.from_numpy(zs).cuda()].cpu().numpy()
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(a))
    world, NL = 8, (1 << n) // 8
    for r in (0, 5):
        loc = ptdr.decompose_zshard(A, "anti_diagonal", r, world)
        assert torch.equal(torch.view_as_real(loc), torch.view_as_real(out[r * NL:(r + 1) * NL]))


@pytest.mark.parametrize("s", [0, 1, 2, 3, 5])
@pytest.mark.parametrize("n", [3, 4, 6, 9, 12])
def test_band_full(gpu, s, n):
    torch = _torch()
    if (1 << n) <= s:
        pytest.skip("band wider than the matrix")
    rng = np.random.default_rng(2000 + 10 * n + s)
    diags = _cplx(rng, (2 * s + 1, 1 << n))
    out = ptdr.decompose_band(torch.from_numpy(diags).cuda(), s).cpu().numpy()
    xs = ptdr.band_xmasks(n, s)
    zs = np.arange(1 << n)
    qs = np.concatenate([_qs_block(x, n, zs) for x in xs])
    want = oracle.coeffs_band(diags, s, qs)
    err = np.max(np.abs(out - want))
    assert err <= TOL * np.max(np.abs(diags)), err
    assert ptdr.last_launch_count() >= 2


def test_band_outside_support_is_zero(gpu):
    """Strings outside the returned X-mask blocks have coefficient exactly 0 (oracle)."""
    n, s = 7, 3
    rng = np.random.default_rng(77)
    diags = _cplx(rng, (2 * s + 1, 1 << n))
    xs = set(ptdr.band_xmasks(n, s).tolist())
    others = [x for x in range(1 << n) if x not in xs]
    qs = np.array([q_of(x, int(z), n) for x in others[::5] for z in rng.integers(0, 1 << n, 4)], dtype=np.uint64)
    assert np.all(oracle.coeffs_band(diags, s, qs) == 0)


@pytest.mark.parametrize("structure,s", [("diagonal", 0), ("tridiagonal", 1)])
def test_band_matches_structured_paths(gpu, structure, s):
    """s = 0 / s = 1 through the general band planner == the DIAGONAL / TRIDIAGONAL paths."""
    torch = _torch()
    n = 14
    B = ptdr.generate_band(n, 3, structure)
    ref = ptdr.decompose(B, structure)
    N = 1 << n
    if structure == "diagonal":
        diags = B.view(1, N)
    else:
        sub, main, sup = B.view(3, N)
        # TRIDIAGONAL storage: sub[i] = A[i][i-1], main[i] = A[i][i], sup[i] = A[i][i+1],
        # which is exactly diags[d + 1][i] = A[i][i + d]
        diags = torch.stack([sub, main, sup])
    got = ptdr.decompose_band(diags.contiguous(), s)
    assert torch.max(torch.abs(got - ref)).item() <= TOL * torch.max(torch.abs(B)).item()


def test_band_n20_sampled(gpu):
    torch = _torch()
    n, s = 20, 2
    rng = np.random.default_rng(20)
    diags = _cplx(rng, (2 * s + 1, 1 << n))
    out = ptdr.decompose_band(torch.from_numpy(diags).cuda(), s)
    xs = ptdr.band_xmasks(n, s)
    b = rng.integers(0, len(xs), 1500)
    z = rng.integers(0, 1 << n, 1500)
    qs = np.array([q_of(int(xs[i]), int(zz), n) for i, zz in zip(b, z)], dtype=np.uint64)
    want = oracle.coeffs_band(diags, s, qs)
    got = out[torch.from_numpy(b * (1 << n) + z).cuda()].cpu().numpy()
    assert np.max(np.abs(got - want)) <= TOL * np.max(np.abs(diags))


@pytest.mark.parametrize("n,s", [(14, 1), (15, 3), (16, 17), (17, 64)])
def test_band_top_levels_gather(gpu, n, s):
    """n >= 14: the gather runs the top butterfly levels of every long segment (three, four for
    x = 0) and scatters the short segments and the rows whose + d crosses a top-block boundary
    one by one (band.cu band_gather_top3_kernel); sampled against the oracle in every block,
    with the strings of the last rows of each top block included."""
    torch = _torch()
    rng = np.random.default_rng(4000 + n + s)
    diags = _cplx(rng, (2 * s + 1, 1 << n))
    out = ptdr.decompose_band(torch.from_numpy(diags).cuda(), s).cpu().numpy().reshape(-1, 1 << n)
    xs = ptdr.band_xmasks(n, s)
    N = 1 << n
    bs = np.concatenate([np.arange(len(xs)), rng.integers(0, len(xs), 1500)])
    zs = np.concatenate([np.full(len(xs), N - 1), rng.integers(0, N, 1500)])
    qs = np.array([q_of(int(xs[b]), int(z), n) for b, z in zip(bs, zs)], dtype=np.uint64)
    want = oracle.coeffs_band(diags, s, qs)
    err = np.max(np.abs(out[bs, zs] - want))
    assert err <= TOL * np.max(np.abs(diags)), err
    # Parseval over all blocks: sum |alpha|^2 = ||A||_F^2 / 2^n (entries inside the matrix only)
    fro2 = sum(float(np.sum(np.abs(diags[d + s, max(0, -d):N - max(0, d)]) ** 2)) for d in range(-s, s + 1))
    assert abs(float(np.sum(np.abs(out) ** 2)) - fro2 / N) <= 1e-11 * fro2 / N


@pytest.mark.parametrize("n,s,full", [(9, 17, True), (10, 33, False), (12, 64, False)])
def test_band_wide(gpu, n, s, full):
    """Wide bands: blocks with more than 8 segments (|L_x| = #m * 2^popcount(e), e = 2^{t+1}-1-x
    up to s-1) take the expansion's per-segment fallback after its batched first 8."""
    torch = _torch()
    rng = np.random.default_rng(3000 + n + s)
    diags = _cplx(rng, (2 * s + 1, 1 << n))
    out = ptdr.decompose_band(torch.from_numpy(diags).cuda(), s).cpu().numpy().reshape(-1, 1 << n)
    xs = ptdr.band_xmasks(n, s)
    if full:
        bs = np.repeat(np.arange(len(xs)), 1 << n)
        zs = np.tile(np.arange(1 << n), len(xs))
    else:
        bs = rng.integers(0, len(xs), 3000)
        zs = rng.integers(0, 1 << n, 3000)
    qs = np.array([q_of(int(xs[b]), int(z), n) for b, z in zip(bs, zs)], dtype=np.uint64)
    want = oracle.coeffs_band(diags, s, qs)
    err = np.max(np.abs(out[bs, zs] - want))
    assert err <= TOL * np.max(np.abs(diags)), err
