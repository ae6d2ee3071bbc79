"""Guard-band memory checks of every kernel family (our own bounds checking: the pool's
compute-sanitizer is closed).

Every device buffer a call touches -- inputs, output, workspace -- is a view in the middle
of a larger allocation whose 64 KiB guard bands on both sides hold a NaN bit pattern
(complex128) or 0xA5 bytes (workspace).  The output view itself is prefilled with the NaN
pattern.  After the call:
  * both guard bands of every buffer are bit-identical to the pattern (no out-of-bounds
    write, before or after, by any kernel of the call);
  * the output is bit-identical to the same call on ordinary allocations -- an
    out-of-bounds read would pull a NaN from a guard band into some coefficient, and an
    output element the call never wrote would still hold the NaN pattern.
Sizes span the kernel families: whole-vector tiles (n <= 10), the fused two-phase pipeline
(n >= 11), ragged shard widths, the band paths and their z-shards, the batched, padded,
generated, peer and algebra entry points, and the generators."""
import numpy as np
import pytest

import paper_2403_11644_b200 as ptdr

pytestmark = pytest.mark.gpu

G = 4096                      # guard elements per side (64 KiB of complex128)
NAN_BITS = 0x7FF4DEADBEEF0001  # a signalling-NaN payload no kernel produces
BYTE = 0xA5


def _torch():
    import torch

    return torch


class Arena:
    """Guarded views; check() verifies every guard band."""

    def __init__(self):
        self.bufs = []

    def c128(self, count, like=None):
        torch = _torch()
        buf = torch.empty(count + 2 * G, dtype=torch.complex128, device="cuda")
        torch.view_as_real(buf).view(torch.int64).fill_(NAN_BITS)
        view = buf[G:G + count]
        if like is not None:
            view.copy_(like.reshape(-1))
        self.bufs.append(("c", buf, count))
        return view

    def i64(self, count, like):
        torch = _torch()
        buf = torch.full((count + 2 * G,), NAN_BITS, dtype=torch.int64, device="cuda")
        view = buf[G:G + count]
        view.copy_(like)
        self.bufs.append(("i", buf, count))
        return view

    def ws(self, nbytes):
        torch = _torch()
        nb = max(int(nbytes), 1)
        buf = torch.full((nb + 2 * G * 16,), BYTE, dtype=torch.uint8, device="cuda")
        self.bufs.append(("b", buf, nb))
        return buf[G * 16:G * 16 + nb]

    def check(self):
        torch = _torch()
        torch.cuda.synchronize()
        for kind, buf, count in self.bufs:
            if kind == "c":
                bits = torch.view_as_real(buf).view(torch.int64).reshape(-1, 2)
                lo, hi = bits[:G], bits[G + count:]
                assert bool((lo == NAN_BITS).all()), "write below a complex128 buffer"
                assert bool((hi == NAN_BITS).all()), "write above a complex128 buffer"
            elif kind == "i":
                assert bool((buf[:G] == NAN_BITS).all()) and bool((buf[G + count:] == NAN_BITS).all()), \
                    "write around an int64 buffer"
            else:
                lo, hi = buf[:G * 16], buf[G * 16 + count:]
                assert bool((lo == BYTE).all()), "write below a workspace"
                assert bool((hi == BYTE).all()), "write above a workspace"


def _bits(t):
    torch = _torch()
    return torch.view_as_real(t.reshape(-1)).view(torch.int64)


def _same(got, want):
    torch = _torch()
    assert bool(torch.isfinite(torch.view_as_real(got)).all()), "NaN pattern in the output"
    assert torch.equal(_bits(got), _bits(want)), "differs from the unguarded call"


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 8, 9, 10, 11, 12, 13, 14])
@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
def test_dense_guarded(gpu, n, variant):
    if n == 14 and variant != "general":
        pytest.skip("one n=14 variant is enough (4 GiB buffers)")
    N = 1 << n
    A0 = ptdr.generate_dense(n, 11, variant)
    want = ptdr.decompose(A0, variant)
    ar = Arena()
    A = ar.c128(N * N, A0).view(N, N)
    out = ar.c128(4 ** n)
    ws = ar.ws(ptdr.workspace_bytes(n, variant))
    ptdr.decompose(A, variant, out=out, workspace=ws)
    ar.check()
    _same(out, want)


@pytest.mark.parametrize("structure", ["diagonal", "tridiagonal", "anti_diagonal", "hermitian_tridiagonal"])
@pytest.mark.parametrize("n", [1, 2, 4, 8, 9, 12, 14, 17])
def test_band_structures_guarded(gpu, structure, n):
    torch = _torch()
    N = 1 << n
    rows = {"tridiagonal": 3, "hermitian_tridiagonal": 2}.get(structure, 1)
    rng = np.random.default_rng(n)
    b0 = torch.from_numpy(rng.standard_normal((rows, N)) + 1j * rng.standard_normal((rows, N))).cuda()
    if rows == 1:
        b0 = b0[0].contiguous()
    want = ptdr.decompose(b0, structure)
    ar = Arena()
    b = ar.c128(rows * N, b0).view(b0.shape)
    out = ar.c128(ptdr.output_count(n, structure))
    ws = ar.ws(ptdr.workspace_bytes(n, structure))
    ptdr.decompose(b, structure, out=out, workspace=ws)
    ar.check()
    _same(out, want)
    for world in (2, 4):   # z-sharded: every rank's slice guarded separately
        if N % world or N // world < 1:
            continue
        full = ptdr.output_count(n, structure)
        blocks = full // N
        got = torch.empty(full, dtype=torch.complex128, device="cuda").view(blocks, N)
        for r in range(world):
            ar = Arena()
            o = ar.c128(full // world)
            w = ar.ws(ptdr.workspace_bytes(n, structure, world))
            ptdr.decompose_zshard(b0, structure, r, world, out=o, workspace=w)
            ar.check()
            Z = N // world
            got[:, r * Z:(r + 1) * Z] = o.view(blocks, Z)
        _same(got.reshape(-1), want)


@pytest.mark.parametrize("n,s", [(3, 1), (6, 2), (10, 3), (12, 2)])
def test_band_s_guarded(gpu, n, s):
    torch = _torch()
    N = 1 << n
    rng = np.random.default_rng(100 + n)
    d0 = torch.from_numpy(rng.standard_normal((2 * s + 1, N)) + 1j * rng.standard_normal((2 * s + 1, N))).cuda()
    want = ptdr.decompose_band(d0, s)
    ar = Arena()
    d = ar.c128(d0.numel(), d0).view(d0.shape)
    out = ar.c128(want.numel())
    ws = ar.ws(ptdr.lib().ptdr_band_workspace_bytes(n, s))
    ptdr.decompose_band(d, s, out=out, workspace=ws)
    ar.check()
    _same(out, want)


@pytest.mark.parametrize("n,world", [(6, 2), (9, 4), (12, 2), (13, 4)])
def test_xshard_guarded(gpu, n, world):
    torch = _torch()
    N, R = 1 << n, (1 << n) // world
    for h in (0, world - 1):
        recv0 = torch.randn(N * R, dtype=torch.complex128, device="cuda")
        want = ptdr.decompose_xshard(recv0.view(N, R), n, h, world)
        ar = Arena()
        recv = ar.c128(N * R, recv0).view(N, R)
        out = ar.c128(4 ** n // world)
        ws = ar.ws(ptdr.workspace_bytes(n, "general", world))
        ptdr.decompose_xshard(recv, n, h, world, out=out, workspace=ws)
        ar.check()
        _same(out, want)


@pytest.mark.parametrize("n,world", [(12, 2), (13, 4)])
def test_peer_guarded(gpu, n, world):
    N, R = 1 << n, (1 << n) // world
    A0 = ptdr.generate_dense(n, 5, "general")
    ar = Arena()
    shards = [ar.c128(R * N, A0[r * R:(r + 1) * R]) for r in range(world)]
    ptrs = [s.data_ptr() for s in shards]
    for h in (0, world - 1):
        plain = [A0[r * R:(r + 1) * R].clone() for r in range(world)]   # ordinary allocations
        want = ptdr.decompose_peer([p.data_ptr() for p in plain], n, h, world)
        out = ar.c128(4 ** n // world)
        ws = ar.ws(ptdr.workspace_bytes(n, "general", world))
        ptdr.decompose_peer(ptrs, n, h, world, out=out, workspace=ws)
        ar.check()
        _same(out, want)


@pytest.mark.parametrize("m,pitch", [(1, 1), (5, 7), (100, 100), (1000, 1003), (2100, 2100)])
def test_padded_guarded(gpu, m, pitch):
    torch = _torch()
    n = max(1, (m - 1).bit_length())
    full0 = torch.randn(m * pitch, dtype=torch.complex128, device="cuda")
    A0 = full0.view(m, pitch)[:, :m]
    want = ptdr.decompose_padded(A0)
    ar = Arena()
    full = ar.c128(m * pitch, full0)
    A = full.view(m, pitch)[:, :m]
    out = ar.c128(4 ** n)
    ws = ar.ws(ptdr.lib().ptdr_padded_workspace_bytes(m, 0))
    ptdr.decompose_padded(A, out=out, workspace=ws)
    ar.check()
    _same(out, want)


@pytest.mark.parametrize("n,batch", [(1, 3), (3, 5), (6, 7), (9, 3), (10, 2)])
@pytest.mark.parametrize("variant", ["general", "hermitian"])
def test_batched_guarded(gpu, n, batch, variant):
    torch = _torch()
    N = 1 << n
    A0 = torch.stack([ptdr.generate_dense(n, 20 + b, variant) for b in range(batch)]).contiguous()
    want = ptdr.decompose_batched(A0, variant)
    ar = Arena()
    A = ar.c128(A0.numel(), A0).view(batch, N, N)
    out = ar.c128(batch * 4 ** n).view(batch, 4 ** n)
    ptdr.decompose_batched(A, variant, out=out)
    ar.check()
    _same(out, want)


@pytest.mark.parametrize("n", [1, 6, 11])
def test_coefficients_guarded(gpu, n):
    torch = _torch()
    N = 1 << n
    A0 = ptdr.generate_dense(n, 3, "general")
    rng = np.random.default_rng(n)
    q0 = torch.from_numpy(rng.integers(0, 4 ** n, size=777, dtype=np.int64)).cuda()
    want = ptdr.coefficients(A0, q0)
    ar = Arena()
    A = ar.c128(N * N, A0).view(N, N)
    q = ar.i64(q0.numel(), q0)   # an out-of-range read would fetch a guard word as a q index
    out = ar.c128(q0.numel())
    ptdr.coefficients(A, q, out=out)
    ar.check()
    _same(out, want)


@pytest.mark.parametrize("n,world", [(4, 1), (11, 1), (12, 2), (13, 4)])
def test_generated_guarded(gpu, n, world):
    for r in {0, world - 1}:
        want = ptdr.decompose_generated(n, 7, r, world)
        ar = Arena()
        out = ar.c128(4 ** n // world)
        ws = ar.ws(ptdr.lib().ptdr_generated_workspace_bytes(n, world))
        ptdr.decompose_generated(n, 7, r, world, out=out, workspace=ws)
        ar.check()
        _same(out, want)


@pytest.mark.parametrize("n", [1, 4, 8, 9, 11, 12])
def test_reconstruct_guarded(gpu, n):
    N = 1 << n
    c0 = ptdr.decompose(ptdr.generate_dense(n, 2, "general"))
    want = ptdr.reconstruct(c0)
    ar = Arena()
    c = ar.c128(4 ** n, c0)
    out = ar.c128(N * N).view(N, N)
    ws = ar.ws(ptdr.lib().ptdr_reconstruct_workspace_bytes(n))
    ptdr.reconstruct(c, out=out, workspace=ws)
    ar.check()
    _same(out, want)


@pytest.mark.parametrize("n", [3, 8, 11, 12])
def test_reconstruct_matrix_layout_guarded(gpu, n):
    """The inverse from the matrix layout (MODE_INV pipeline from n = 11), out of place and in
    place, writes nothing outside its buffers."""
    N = 1 << n
    M0 = ptdr.decompose_matrix_layout(ptdr.generate_dense(n, 3, "general"))
    want = ptdr.reconstruct_matrix_layout(M0)
    ar = Arena()
    M = ar.c128(N * N, M0).view(N, N)
    out = ar.c128(N * N).view(N, N)
    ws = ar.ws(ptdr.lib().ptdr_reconstruct_matrix_layout_workspace_bytes(n))
    ptdr.reconstruct_matrix_layout(M, out=out, workspace=ws)
    ar.check()
    _same(out, want)
    ar = Arena()
    M = ar.c128(N * N, M0).view(N, N)
    ws = ar.ws(ptdr.lib().ptdr_reconstruct_matrix_layout_workspace_bytes(n))
    ptdr.reconstruct_matrix_layout(M, workspace=ws, inplace=True)
    ar.check()
    _same(M, want)


def test_algebra_guarded(gpu):
    torch = _torch()
    x0 = torch.randn(1001, dtype=torch.complex128, device="cuda")
    y0 = torch.randn(1001, dtype=torch.complex128, device="cuda")
    want = ptdr.axpby(0.5 - 2j, x0, 1.5j, y0)
    ar = Arena()
    x, y, out = ar.c128(1001, x0), ar.c128(1001, y0), ar.c128(1001)
    ptdr.axpby(0.5 - 2j, x, 1.5j, y, out=out)
    ar.check()
    _same(out, want)
    for n, k in [(1, 1), (3, 2), (5, 1), (2, 4)]:
        b0 = torch.randn(1 << k, 4 ** n, dtype=torch.complex128, device="cuda")
        want = ptdr.block_diag(b0)
        ar = Arena()
        b = ar.c128(b0.numel(), b0).view(b0.shape)
        out = ar.c128(4 ** (n + k))
        ptdr.block_diag(b, out=out)
        ar.check()
        _same(out, want)
    for n in (1, 5, 9):
        c0 = torch.randn(4 ** n, dtype=torch.complex128, device="cuda")
        want = ptdr.hermitian_augment(c0)
        ar = Arena()
        c, out = ar.c128(4 ** n, c0), ar.c128(4 ** (n + 1))
        ptdr.hermitian_augment(c, out=out)
        ar.check()
        _same(out, want)


@pytest.mark.parametrize("n", [1, 5, 10, 13])
def test_generators_guarded(gpu, n):
    N = 1 << n
    for variant in ("general", "hermitian", "real_symmetric"):
        want = ptdr.generate_dense(n, 9, variant)
        ar = Arena()
        out = ar.c128(N * N).view(N, N)
        ptdr.generate_dense(n, 9, variant, out=out)
        ar.check()
        _same(out, want)
    if n >= 2:   # a row block
        R = N // 2
        want = ptdr.generate_dense(n, 9, "general", row0=R, nrows=R)
        ar = Arena()
        out = ar.c128(R * N).view(R, N)
        ptdr.generate_dense(n, 9, "general", row0=R, nrows=R, out=out)
        ar.check()
        _same(out, want)
    for variant in ("diagonal", "tridiagonal"):
        want = ptdr.generate_band(n, 9, variant)
        ar = Arena()
        out = ar.c128(want.numel()).view(want.shape)
        ptdr.generate_band(n, 9, variant, out=out)
        ar.check()
        _same(out, want)


def test_guard_harness_detects(gpu):
    """The harness itself: a write one element past a view fails check(), and one
    guard-pattern word read as input reaches the output as a non-finite coefficient."""
    torch = _torch()
    ar = Arena()
    v = ar.c128(100)
    full = v.as_strided((101,), (1,))   # one past the end
    full[100] = 0
    with pytest.raises(AssertionError):
        ar.check()
    n, N = 11, 1 << 11
    A0 = ptdr.generate_dense(n, 11, "general")
    ar = Arena()
    A = ar.c128(N * N, A0).view(N, N)
    torch.view_as_real(A)[N - 1, N - 1].view(torch.int64).fill_(NAN_BITS)
    out = ptdr.decompose(A)
    assert not bool(torch.isfinite(torch.view_as_real(out)).all())
