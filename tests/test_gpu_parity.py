"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Tolerance (BASELINE.json north_star): |alpha_gpu - alpha_oracle| <= 1e-12 * max|A_ij|
per coefficient (complex modulus).  Inputs are seeded and synthetic
(ptdr_inputs); the oracle never sees a value produced by the CUDA path.
"""
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


def _gpu_decompose(A_host, structure="general"):
    torch = _torch()
    A = torch.from_numpy(np.ascontiguousarray(A_host)).cuda()
    out = ptdr.decompose(A, structure)
    torch.cuda.synchronize()
    assert ptdr.last_launch_count() >= 1
    return out.cpu().numpy()


def _assert_close(got, want, maxabs, what=""):
    err = np.max(np.abs(got - want)) if got.size else 0.0
    assert err <= TOL * maxabs, f"{what}: max err {err:.3e} > {TOL * maxabs:.3e}"


def _dense(n, seed, variant):
    return ptdr_inputs.dense(n, seed, variant)


# ---------------------------------------------------------------- full-oracle sweeps
@pytest.mark.parametrize("n", list(range(1, 11)))
@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_dense_full_oracle(gpu, n, variant):
    A = _dense(n, 100 + n, variant)
    got = _gpu_decompose(A, variant)
    want = oracle.decompose(A)
    _assert_close(got, want, np.max(np.abs(A)), f"n={n} {variant}")
    if variant != "general":
        assert np.all(got.imag == 0)          # HERMITIAN / REAL_SYMMETRIC write Im = 0 exactly


@pytest.mark.parametrize("n", [11, 12, 13, 14])
@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_dense_sampled_oracle(gpu, n, variant):
    A = _dense(n, 200 + n, variant)
    got = _gpu_decompose(A, variant)
    rng = np.random.default_rng(n)
    qs = np.unique(np.concatenate([rng.integers(0, 4 ** n, 1500), _edge_qs(n)])).astype(np.uint64)
    want = oracle.coeffs_dense(A, qs)
    _assert_close(got[qs.astype(np.int64)], want, np.max(np.abs(A)), f"n={n} {variant}")
    # Parseval (Theorem 1): sum |alpha|^2 = ||A||_F^2 / 2^n
    lhs = np.sum(np.abs(got) ** 2)
    rhs = oracle.frobenius2(A) / (1 << n)
    assert abs(lhs - rhs) / rhs < 1e-11


def _edge_qs(n):
    """I^n, X^n, Y^n, Z^n, single letters at both ends, last q."""
    qs = [0, 4 ** n - 1]
    for code in (1, 2, 3):
        qs.append(sum(code << (2 * l) for l in range(n)))
        qs.append(code)
        qs.append(code << (2 * (n - 1)))
    return np.array(qs, dtype=np.int64)


# ---------------------------------------------------------------- closed forms / edge cases
@pytest.mark.parametrize("n", [1, 3, 6, 9, 12])
def test_identity_one_hot(gpu, n):
    got = _gpu_decompose(np.eye(1 << n, dtype=np.complex128))
    assert got[0] == 1.0 and np.count_nonzero(got) == 1


@pytest.mark.parametrize("n", [2, 5, 8, 11])
def test_single_string_one_hot(gpu, n):
    from tests.paulis import kron_string

    rng = np.random.default_rng(n)
    for q0 in list(rng.integers(0, 4 ** n, 2)) + [4 ** n - 1]:
        P = kron_string(oracle.string_of(int(q0), n))
        got = _gpu_decompose(P)
        assert got[q0] == 1.0 and np.count_nonzero(got) == 1


@pytest.mark.parametrize("n", [4, 9, 12])
def test_cross_structure_paths(gpu, n):
    A = _dense(n, 7, "hermitian")
    g = _gpu_decompose(A, "general")
    h = _gpu_decompose(A, "hermitian")
    _assert_close(h, g, np.max(np.abs(A)), "hermitian vs general")
    S = _dense(n, 7, "real_symmetric")
    _assert_close(_gpu_decompose(S, "real_symmetric"), _gpu_decompose(S, "general"),
                  np.max(np.abs(S)), "real_symmetric vs general")


@pytest.mark.parametrize("n", [1, 2, 4, 7, 10, 12])
def test_band_paths_vs_dense(gpu, n):
    d = ptdr_inputs.band(n, 30 + n, "diagonal")
    got = _gpu_decompose(d, "diagonal")
    dense = _gpu_decompose(np.diag(d), "general")
    qs = [ptdr.q_of(0, z, n) for z in range(1 << n)]
    _assert_close(got, dense[qs], np.max(np.abs(d)), "diagonal")
    sub, main, sup = ptdr_inputs.band(n, 40 + n, "tridiagonal")
    # complex, non-symmetric tridiagonal exercises S_t != U_t
    rng = np.random.default_rng(n)
    sub = sub + 1j * rng.standard_normal(sub.shape)
    sup = sup + 0.5 * rng.standard_normal(sup.shape)
    sub[0] = 0
    sup[-1] = 0
    band = np.stack([sub, main, sup])
    got = _gpu_decompose(band, "tridiagonal").reshape(n + 1, 1 << n)
    Ad = ptdr_inputs.densify_band(n, main, sub, sup)
    dense = _gpu_decompose(Ad, "general")
    for b in range(n + 1):
        x = (1 << b) - 1
        qs = [ptdr.q_of(x, z, n) for z in range(1 << n)]
        _assert_close(got[b], dense[qs], np.max(np.abs(band)), f"tridiagonal block {b}")
    # Table I (l.513): everything outside the n+1 blocks is zero
    inblock = {ptdr.q_of((1 << b) - 1, z, n) for b in range(n + 1) for z in range(1 << n)}
    outside = np.array([q for q in range(4 ** n) if q not in inblock], dtype=np.int64)
    if outside.size:
        assert np.max(np.abs(dense[outside])) <= TOL * np.max(np.abs(band))


@pytest.mark.parametrize("n", [3, 8, 11])
def test_band_oracle(gpu, n):
    sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
    got = _gpu_decompose(np.stack([sub, main, sup]), "tridiagonal").reshape(n + 1, 1 << n)
    for b in range(n + 1):
        x = (1 << b) - 1
        qs = np.array([ptdr.q_of(x, z, n) for z in range(1 << n)], dtype=np.uint64)
        want = oracle.coeffs_tridiagonal(sub, main, sup, qs)
        _assert_close(got[b], want, np.max(np.abs(main)) + np.max(np.abs(sup)), f"block {b}")
    d = ptdr_inputs.band(n, 3, "diagonal")
    got = _gpu_decompose(d, "diagonal")
    qs = np.array([ptdr.q_of(0, z, n) for z in range(1 << n)], dtype=np.uint64)
    _assert_close(got, oracle.coeffs_diagonal(d, qs), np.max(np.abs(d)), "diagonal")


def test_determinism_bitwise(gpu):
    A = _dense(12, 5, "general")
    a = _gpu_decompose(A)
    b = _gpu_decompose(A)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("n,variant,reps", [(11, "general", 200), (13, "hermitian", 100), (15, "general", 10)])
def test_pipeline_repeatable_under_stress(gpu, n, variant, reps):
    """The pipeline's inter-CTA hand-offs (dependency counters, scratch ring, discards) must
    not race: many back-to-back launches reproduce the first result bit for bit."""
    import torch

    A = ptdr.generate_dense(n, 4, variant)
    ws = ptdr.alloc_workspace(n, variant, 1, "cuda")
    ref = ptdr.decompose(A, variant, workspace=ws).clone()
    out = torch.empty_like(ref)
    for _ in range(reps):
        out.fill_(float("nan"))
        ptdr.decompose(A, variant, out=out, workspace=ws)
        assert torch.equal(torch.view_as_real(out).view(torch.int64), torch.view_as_real(ref).view(torch.int64))


def test_host_entry_point(gpu):
    A = _dense(9, 9, "general")
    got = ptdr.decompose_host(A)
    _assert_close(got, oracle.decompose(A), np.max(np.abs(A)), "decompose_host")


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_host_plan_stream(gpu, depth):
    """ptdr_plan_*: a stream of distinct host matrices through `depth` device slots; every
    result equals the oracle (slot reuse must never mix up inputs and outputs)."""
    torch = _torch()
    n, mats = 9, 5
    As = [_dense(n, 20 + k, "general") for k in range(mats)]
    hin = [torch.from_numpy(a).pin_memory() for a in As]
    hout = [torch.empty(4 ** n, dtype=torch.complex128).pin_memory() for _ in range(mats)]
    with ptdr.HostPlan(n, "general", depth=depth) as plan:
        for k in range(mats):
            plan.decompose_async(hin[k], hout[k])
        plan.wait()
        assert plan.launch_count() >= 1
    for k in range(mats):
        _assert_close(hout[k].numpy(), oracle.decompose(As[k]), np.max(np.abs(As[k])), f"plan[{k}]")


def test_host_plan_structures(gpu):
    torch = _torch()
    n = 8
    H = _dense(n, 3, "hermitian")
    out = np.empty(4 ** n, dtype=np.complex128)
    with ptdr.HostPlan(n, "hermitian", depth=1) as plan:
        plan.decompose_async(np.ascontiguousarray(H), out)
        plan.wait()
    _assert_close(out, oracle.decompose(H), np.max(np.abs(H)), "plan hermitian")
    with pytest.raises(ptdr.PtdrError):
        ptdr.HostPlan(n, "general", depth=0)
    with pytest.raises(ValueError):
        with ptdr.HostPlan(n, "general", depth=1) as plan:
            plan.decompose_async(np.zeros(16, np.complex128), out)


def test_error_paths(gpu):
    torch = _torch()
    A = torch.zeros((256, 256), dtype=torch.complex128, device="cuda")
    with pytest.raises(ptdr.PtdrError) as e:
        ptdr.decompose(A, out=A.view(-1))                # out aliases A
    assert e.value.status == ptdr.PTDR_EUNSUPPORTED
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        ptdr.decompose(A, workspace=ws)                  # the binding checks the size first
    out = torch.empty(4 ** 8, dtype=torch.complex128, device="cuda")
    import ctypes
    st = ptdr.lib().ptdr_decompose_async(ctypes.c_void_p(A.data_ptr()), 8, 0, ctypes.c_void_p(out.data_ptr()),
                                         ctypes.c_void_p(ws.data_ptr()), 16, None)
    assert st == ptdr.PTDR_ENOMEM                        # ... and so does the ABI
    with pytest.raises(TypeError):
        ptdr.decompose(A.cpu())                          # no CPU fallback


@pytest.mark.parametrize("n", [1, 6, 11, 13])
@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_zero_matrix_gives_exact_zeros(gpu, n, variant):
    """Degenerate input: A = 0 decomposes to exactly 0 on every path (no stale scratch,
    no uninitialised output)."""
    torch = _torch()
    A = torch.zeros((1 << n, 1 << n), dtype=torch.complex128, device="cuda")
    out = torch.full((4 ** n,), complex(float("nan"), float("nan")), dtype=torch.complex128, device="cuda")
    ptdr.decompose(A, variant, out=out)
    assert torch.count_nonzero(torch.view_as_real(out)).item() == 0


@pytest.mark.parametrize("n", [1, 3, 8, 12])
def test_selected_coefficients_vs_oracle(gpu, n):
    """ptdr_coefficients_async (Algorithm 2 per string on the GPU) vs the oracle."""
    torch = _torch()
    A = _dense(n, 300 + n, "general")
    rng = np.random.default_rng(300 + n)
    qs = np.unique(np.concatenate([rng.integers(0, 4 ** n, 300), _edge_qs(n)])).astype(np.int64)
    got = ptdr.coefficients(torch.from_numpy(A).cuda(), torch.from_numpy(qs).cuda()).cpu().numpy()
    want = oracle.coeffs_dense(A, qs.astype(np.uint64))
    _assert_close(got, want, np.max(np.abs(A)), f"coefficients n={n}")


def test_selected_coefficients_n15_match_transform(gpu):
    """At the bench size: the direct per-string evaluation agrees with the full transform."""
    torch = _torch()
    n = 15
    A = ptdr.generate_dense(n, 4, "general")
    full = ptdr.decompose(A)
    rng = np.random.default_rng(15)
    qs = torch.from_numpy(rng.integers(0, 4 ** n, 512).astype(np.int64)).cuda()
    got = ptdr.coefficients(A, qs)
    err = torch.max(torch.abs(got - full[qs])).item()
    assert err <= TOL * 6.0, err
    del A, full
    torch.cuda.empty_cache()
