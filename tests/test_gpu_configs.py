"""GPU parity at BASELINE.json's configurations, in the launch configuration
bench.py times (device-generated input, ptdr_decompose_async on the current
stream).  Large n: 4096 seeded sampled coefficients vs the oracle (entries
regenerated on the host by the independent input module) + Parseval.
Also the X-mask sharded path, emulated rank by rank on one GPU (independent
launches; no inter-rank waiting)."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs
from paper_2403_11644_b200 import dist as pdist

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _torch():
    import torch

    return torch


def _sample_qs(n, count=4096, seed=1000):
    # fixed edge strings + mt19937_64-style seeded draws
    rng = np.random.default_rng(seed + n)
    edge = [0, 4 ** n - 1]
    for code in (1, 2, 3):
        edge += [sum(code << (2 * l) for l in range(n)), code, code << (2 * (n - 1))]
    q = np.concatenate([np.array(edge, dtype=np.uint64),
                        rng.integers(0, 4 ** n, count - len(edge), dtype=np.uint64)])
    return q


def _sumsq(t):
    """sum |t|^2 in float64, chunked so no large temporaries are allocated."""
    torch = _torch()
    flat = torch.view_as_real(t.reshape(-1))
    total = 0.0
    step = 1 << 26
    for i in range(0, flat.shape[0], step):
        c = flat[i:i + step]
        total += torch.sum(c * c).item()
    return total


def _parseval_gpu(A, out, n):
    lhs = _sumsq(out)
    rhs = _sumsq(A) / (1 << n)
    return abs(lhs - rhs) / rhs


@pytest.mark.parametrize("cfg", [("n6", 6, 0, "general"), ("n10a", 10, 1, "general"),
                                 ("n10b", 10, 1, "hermitian")])
def test_small_configs_full_oracle(gpu, cfg):
    torch = _torch()
    _, n, seed, variant = cfg
    A = ptdr.generate_dense(n, seed, variant)
    out = ptdr.decompose(A, variant).cpu().numpy()
    Ah = ptdr_inputs.dense(n, seed, variant)          # host regeneration (independent)
    want = oracle.decompose(Ah)
    assert np.max(np.abs(out - want)) <= TOL * np.max(np.abs(Ah))
    if variant == "hermitian":
        assert np.all(out.imag == 0)
    del A
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [("n13a", 13, 2, "hermitian"), ("n13b", 13, 2, "real_symmetric"),
                                 ("n15", 15, 4, "general"), ("n16", 16, 4, "general"),
                                 ("n15h", 15, 4, "hermitian"), ("n15s", 15, 4, "real_symmetric"),
                                 ("n16h", 16, 4, "hermitian")])
def test_large_configs_sampled(gpu, cfg):
    torch = _torch()
    _, n, seed, variant = cfg
    A = ptdr.generate_dense(n, seed, variant)
    out = ptdr.decompose(A, variant)
    torch.cuda.synchronize()
    assert _parseval_gpu(A, out, n) < 1e-11
    maxabs = max(torch.max(torch.abs(A[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    del A
    qs = _sample_qs(n)
    got = out[torch.from_numpy(qs.astype(np.int64)).cuda()].cpu().numpy()
    del out
    torch.cuda.empty_cache()
    want = oracle.coeffs_generated(n, seed, ptdr_inputs.VARIANTS[variant], qs)
    assert np.max(np.abs(got - want)) <= TOL * maxabs
    if variant != "general":
        assert np.all(got.imag == 0)
    if variant == "real_symmetric":
        for q, v in zip(qs, got):
            s = oracle.string_of(int(q), n)
            if s.count("Y") % 2:
                assert v == 0


def _support_x(variant, n, b):
    """X-mask of output block b (include/ptdr.h): tridiagonal 2^b - 1, diagonal 0,
    anti-diagonal 2^n - 1."""
    return {"tridiagonal": (1 << b) - 1, "diagonal": 0, "anti_diagonal": (1 << n) - 1}[variant]


def _outside_support(variant, n, rng, count):
    """(x, z) pairs whose X-mask is NOT an output block: by Table I (l.511/l.513) and the
    anti-diagonal remark (l.391-392) their coefficient is exactly 0."""
    inside = {_support_x(variant, n, b) for b in range(n + 1 if variant == "tridiagonal" else 1)}
    xs = [x for x in (1, 2, 5, (1 << n) - 2, 1 << (n - 1)) if x not in inside]
    while len(xs) < count:
        x = int(rng.integers(0, 1 << n))
        if x not in inside:
            xs.append(x)
    zs = rng.integers(0, 1 << n, len(xs))
    return np.array([ptdr.q_of(int(x), int(z), n) for x, z in zip(xs, zs)], dtype=np.uint64)


@pytest.mark.parametrize("variant", ["tridiagonal", "diagonal", "anti_diagonal"])
def test_n24_band_sampled(gpu, variant):
    """BASELINE configs[3] (n = 24, seed 3): SURVEY 8(c) item 15 -- 4096 seeded in-block
    coefficients against the oracle, 64 out-of-block strings whose oracle value is exactly
    0 (the omitted blocks are the zero blocks), and Parseval over the whole output."""
    torch = _torch()
    n, seed = 24, 3
    gen_variant = "diagonal" if variant == "anti_diagonal" else variant
    band = ptdr.generate_band(n, seed, gen_variant)
    out = ptdr.decompose(band, variant)
    torch.cuda.synchronize()
    # ||A||_F^2 = sum over the stored band (tridiagonal: sub, main and sup, whose unused
    # ends sub[0] and sup[2^n - 1] the generator writes as 0)
    rel = abs(_sumsq(out) - _sumsq(band) / (1 << n)) / (_sumsq(band) / (1 << n))
    assert rel < 1e-11
    rng = np.random.default_rng(24 + len(variant))
    nb = n + 1 if variant == "tridiagonal" else 1
    blocks = np.concatenate([np.arange(nb), rng.integers(0, nb, 4096 - nb)])
    zs = np.concatenate([np.full(nb, (1 << n) - 1), rng.integers(0, 1 << n, 4096 - nb)])
    idx = blocks * (1 << n) + zs
    got = out[torch.from_numpy(idx.astype(np.int64)).cuda()].cpu().numpy()
    del out, band
    torch.cuda.empty_cache()
    qs = np.array([ptdr.q_of(_support_x(variant, n, int(b)), int(z), n) for b, z in zip(blocks, zs)],
                  dtype=np.uint64)
    qout = _outside_support(variant, n, rng, 64)
    assert qout.size == 64
    if variant == "tridiagonal":
        sub, main, sup = ptdr_inputs.band(n, seed, variant)
        want = oracle.coeffs_tridiagonal(sub, main, sup, qs)
        zero = oracle.coeffs_tridiagonal(sub, main, sup, qout)
        maxabs = max(np.max(np.abs(main)), np.max(np.abs(sup)))
    else:
        d = ptdr_inputs.band(n, seed, "diagonal")
        fn = oracle.coeffs_diagonal if variant == "diagonal" else oracle.coeffs_antidiagonal
        want = fn(d, qs)
        zero = fn(d, qout)
        maxabs = np.max(np.abs(d))
    assert np.max(np.abs(got - want)) <= TOL * maxabs
    assert np.all(zero == 0)


@pytest.mark.parametrize("variant", ["hermitian", "real_symmetric"])
def test_n13_complete_xmask_blocks(gpu, variant):
    """BASELINE configs[2] (n = 13, seed 2).  The full oracle over all 4^13 strings takes
    about an hour on 16 host cores (1.8e4-3.3e4 coefficients/s), so
    besides the 4096 samples of test_large_configs_sampled this checks COMPLETE X-mask
    blocks -- every one of the 2^13 Z-masks -- for the X-masks of every kernel regime
    (x = 0 and the mirrored launch's small x, half-length chunks at the top bit boundaries,
    x = 2^13 - 1, and random ones): DESIGN.md reading R19."""
    torch = _torch()
    n, seed = 13, 2
    N = 1 << n
    A = ptdr.generate_dense(n, seed, variant)
    out = ptdr.decompose(A, variant)
    torch.cuda.synchronize()
    maxabs = torch.max(torch.abs(A)).item()
    del A
    rng = np.random.default_rng(1313)
    xs = [0, 1, 15, 16, 31, 32, 1 << 12, (1 << 12) + 1, N - 1] + [int(v) for v in rng.integers(0, N, 3)]
    z = np.arange(N)
    for x in xs:
        qs = np.array([ptdr.q_of(x, int(zz), n) for zz in z], dtype=np.uint64)
        got = out[torch.from_numpy(qs.astype(np.int64)).cuda()].cpu().numpy()
        want = oracle.coeffs_generated(n, seed, ptdr_inputs.VARIANTS[variant], qs)
        assert np.max(np.abs(got - want)) <= TOL * maxabs, x
        assert np.all(got.imag == 0)
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,world", [(10, 2), (10, 4), (12, 8), (8, 2), (6, 4), (11, 2), (13, 8), (14, 4)])
def test_xshard_emulated_bitwise(gpu, n, world):
    """Every rank's shard path on one GPU == the single-GPU result, bit for bit."""
    torch = _torch()
    A = ptdr.generate_dense(n, 4, "general")
    ref = ptdr.decompose(A).cpu().numpy()
    N, R = 1 << n, (1 << n) // world
    sends = [ptdr.generate_sendblocks(n, 4, r, world) for r in range(world)]
    full = np.empty(4 ** n, dtype=np.complex128)
    for h in range(world):
        # emulate the equal-split all-to-all: rank h receives block h of every rank
        recv = torch.stack([sends[g][0, h] for g in range(world)]).contiguous()
        out = ptdr.decompose_xshard(recv.view(N, R), n, h, world).cpu().numpy()
        full[pdist.global_q_array(h, n, world)] = out
    if n >= 8:   # same two-phase schedule on every rank -> bitwise identical
        assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
    else:        # narrow shards use the direct kernel: same values up to rounding
        assert np.max(np.abs(full - ref)) <= TOL * torch.max(torch.abs(A)).item()


@pytest.mark.parametrize("structure", ["diagonal", "tridiagonal", "anti_diagonal"])
@pytest.mark.parametrize("n,world", [(5, 2), (9, 8), (13, 4), (14, 2), (15, 8), (16, 2), (16, 16), (17, 8),
                                     (18, 4), (19, 32)])
def test_zshard_emulated_bitwise(gpu, structure, n, world):
    """Every rank's z-slice (replicated band, no communication) == the same slice of the
    one-GPU output, bit for bit: the long vectors (2^15 elements and up) run their top
    butterfly levels first on every path, a rank keeping only its branches (world <= 8) and
    filtering the rest of its bits in the last pass (world > 8)."""
    torch = _torch()
    B = ptdr.generate_band(n, 3, "diagonal" if structure == "anti_diagonal" else structure)
    ref = ptdr.decompose(B, structure).cpu().numpy()
    blocks = n + 1 if structure == "tridiagonal" else 1
    parts = [ptdr.decompose_zshard(B, structure, r, world).cpu().numpy() for r in range(world)]
    full = pdist.assemble_zshards(parts, n, blocks)
    assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("structure", ["diagonal", "tridiagonal", "anti_diagonal"])
def test_zshard_n24_world8(gpu, structure):
    """BASELINE configs[3] at 8 GPUs: every rank (each independent) vs the one-GPU run."""
    torch = _torch()
    n, world = 24, 8
    B = ptdr.generate_band(n, 3, "diagonal" if structure == "anti_diagonal" else structure)
    ref = ptdr.decompose(B, structure)
    blocks = n + 1 if structure == "tridiagonal" else 1
    NL = (1 << n) // world
    for r in range(world):
        loc = ptdr.decompose_zshard(B, structure, r, world)
        want = ref.view(blocks, 1 << n)[:, r * NL:(r + 1) * NL].reshape(-1)
        assert torch.equal(torch.view_as_real(loc), torch.view_as_real(want)), r
        del loc
    del B, ref
    torch.cuda.empty_cache()
