"""Tridiagonal paths at the sizes where the last P/M pass runs fused with the
expansion (band.cu tri_fused_expand_kernel: segments t <= 3 with 13..20-bit branches, n = 17..24).

The BASELINE n = 24 input is real symmetric (sub[i+1] = sup[i]), so M_t = WHT(S_t - U_t) = 0
there; these inputs make every M_t nonzero and complex.  Checked against the oracle (the
definition Tr(P A)/2^n entry by entry, Sec. IV-A l.395-465) at sampled strings of every
output block incl. the fused ones, exact zeros outside the support (Table I, l.513), Parseval,
and the z-shards at G = 2 / 8 bit for bit against the one-GPU result.

HERMITIAN_TRIDIAGONAL ([main, sup], the sub-diagonal conj(sup) implied) must equal TRIDIAGONAL
on the same matrix bit for bit at every size (the short-segment, top-bits and fused regimes)
and on every z-shard, and match the oracle with exactly real coefficients for a real main
diagonal."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
from paper_2403_11644_b200 import dist as pdist

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _band(n, seed):
    rng = np.random.default_rng(seed)
    N = 1 << n
    sub, main, sup = (rng.standard_normal(N) + 1j * rng.standard_normal(N) for _ in range(3))
    sub[0] = 0.0        # A[0][-1] does not exist
    sup[N - 1] = 0.0    # A[N-1][N] does not exist
    return sub, main, sup


@pytest.mark.parametrize("n", [17, 19, 21])
def test_fused_tridiagonal_vs_oracle(gpu, n):
    import torch

    sub, main, sup = _band(n, 900 + n)
    B = torch.from_numpy(np.stack([sub, main, sup])).cuda()
    out = ptdr.decompose(B, "tridiagonal").cpu().numpy()
    N = 1 << n
    # Parseval: sum |alpha|^2 = ||A||_F^2 / 2^n
    fro2 = sum(float(np.sum(np.abs(v) ** 2)) for v in (sub, main, sup))
    assert abs(float(np.sum(np.abs(out) ** 2)) - fro2 / N) <= 1e-11 * fro2 / N
    rng = np.random.default_rng(n)
    blocks = np.concatenate([np.repeat(np.arange(n + 1), 4), rng.integers(0, n + 1, 384)])
    zs = np.concatenate([np.tile([0, 1, N - 2, N - 1], n + 1), rng.integers(0, N, 384)])
    qs = np.array([ptdr.q_of((1 << int(b)) - 1, int(z), n) for b, z in zip(blocks, zs)], dtype=np.uint64)
    want = oracle.coeffs_tridiagonal(sub, main, sup, qs)
    got = out.reshape(n + 1, N)[blocks, zs]
    maxabs = max(np.max(np.abs(v)) for v in (sub, main, sup))
    assert np.max(np.abs(got - want)) <= TOL * maxabs
    # strings outside the n + 1 X-masks 2^b - 1 are exactly zero
    inside = {(1 << b) - 1 for b in range(n + 1)}
    xo = [x for x in rng.integers(0, N, 64) if int(x) not in inside][:32]
    qo = np.array([ptdr.q_of(int(x), int(z), n) for x, z in zip(xo, rng.integers(0, N, len(xo)))], dtype=np.uint64)
    assert np.all(oracle.coeffs_tridiagonal(sub, main, sup, qo) == 0)
    # the z-sharded path (fused for G <= 8) is the same slice bit for bit
    for world in (2, 8):
        parts = [ptdr.decompose_zshard(B, "tridiagonal", r, world).cpu().numpy() for r in range(world)]
        full = pdist.assemble_zshards(parts, n, n + 1)
        assert np.array_equal(full.view(np.uint64), out.view(np.uint64)), world


def _herm_band(n, seed, complex_main=True):
    rng = np.random.default_rng(seed)
    N = 1 << n
    main = rng.standard_normal(N) + (1j * rng.standard_normal(N) if complex_main else 0.0)
    sup = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    sup[N - 1] = 0.0
    sub = np.zeros(N, dtype=np.complex128)
    sub[1:] = np.conj(sup[:-1])      # A[i+1][i] = conj(A[i][i+1])
    return sub, np.asarray(main, dtype=np.complex128), sup


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 14, 15, 16, 17, 19, 21])
def test_hermitian_tridiagonal_bitwise_equals_general(gpu, n):
    """HERMITIAN_TRIDIAGONAL ([main, sup], sub = conj(sup) implied) == TRIDIAGONAL on the same
    matrix bit for bit (include/ptdr.h: P_t = (2 Re W_t, 0), M_t = (0, 2 Im W_t) are exact),
    on one GPU and on every z-shard of G = 2 / 8."""
    import torch

    sub, main, sup = _herm_band(n, 700 + n)
    G = torch.from_numpy(np.stack([sub, main, sup])).cuda()
    H = torch.from_numpy(np.stack([main, sup])).cuda()
    ref = ptdr.decompose(G, "tridiagonal")
    got = ptdr.decompose(H, "hermitian_tridiagonal")
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))
    for world in (2, 8):
        if world > (1 << n):
            continue
        for r in range(world):
            a = ptdr.decompose_zshard(H, "hermitian_tridiagonal", r, world)
            b = ptdr.decompose_zshard(G, "tridiagonal", r, world)
            assert torch.equal(torch.view_as_real(a), torch.view_as_real(b)), (world, r)


@pytest.mark.parametrize("n", [18, 21])
def test_hermitian_tridiagonal_vs_oracle(gpu, n):
    """Real coefficients (Theorem 2, l.123-136) for a real main diagonal, and the oracle's
    Tr(P A)/2^n at sampled strings of every block."""
    import torch

    sub, main, sup = _herm_band(n, 800 + n, complex_main=False)
    H = torch.from_numpy(np.stack([main, sup])).cuda()
    out = ptdr.decompose(H, "hermitian_tridiagonal").cpu().numpy()
    assert np.all(out.imag == 0)
    N = 1 << n
    rng = np.random.default_rng(n + 5)
    blocks = np.concatenate([np.arange(n + 1), rng.integers(0, n + 1, 255 - n)])
    zs = rng.integers(0, N, blocks.size)
    qs = np.array([ptdr.q_of((1 << int(b)) - 1, int(z), n) for b, z in zip(blocks, zs)], dtype=np.uint64)
    want = oracle.coeffs_tridiagonal(sub, main, sup, qs)
    got = out.reshape(n + 1, N)[blocks, zs]
    maxabs = max(np.max(np.abs(v)) for v in (sub, main, sup))
    assert np.max(np.abs(got - want)) <= TOL * maxabs


def test_hermitian_tridiagonal_generator_and_n24(gpu):
    """The generator's variant 6 is rows [main, sup] of the real symmetric tridiagonal (BASELINE
    configs[3] (a)), its ||A||_F^2 partials count the implied sub-diagonal, and at n = 24 the
    Hermitian path equals the general one bit for bit."""
    import torch

    n, seed = 24, 3
    f_g, f_h = ptdr.fro2_partials(), ptdr.fro2_partials()
    G = ptdr.generate_band(n, seed, "tridiagonal", fro2=f_g)
    H = ptdr.generate_band(n, seed, "hermitian_tridiagonal", fro2=f_h)
    assert torch.equal(torch.view_as_real(H), torch.view_as_real(G[1:3]))
    assert abs(ptdr.fro2_total(f_h) - ptdr.fro2_total(f_g)) <= 1e-12 * ptdr.fro2_total(f_g)
    ref = ptdr.decompose(G, "tridiagonal")
    got = ptdr.decompose(H, "hermitian_tridiagonal")
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))
    del ref, got
    for r in (0, 7):
        a = ptdr.decompose_zshard(H, "hermitian_tridiagonal", r, 8)
        b = ptdr.decompose_zshard(G, "tridiagonal", r, 8)
        assert torch.equal(torch.view_as_real(a), torch.view_as_real(b)), r
    torch.cuda.empty_cache()


def test_hermitian_tridiagonal_host_entry_points(gpu):
    """ptdr_decompose_host and the streaming host plan accept the new structure ([2, 2^n]
    input) and return the device result."""
    import torch

    n = 17
    sub, main, sup = _herm_band(n, 901)
    H = np.ascontiguousarray(np.stack([main, sup]))
    want = ptdr.decompose(torch.from_numpy(H).cuda(), "hermitian_tridiagonal").cpu().numpy()
    got = ptdr.decompose_host(H, "hermitian_tridiagonal")
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    out = np.empty_like(want)
    with ptdr.HostPlan(n, "hermitian_tridiagonal", depth=2) as plan:
        plan.decompose_async(H, out)
        plan.wait()
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))
