"""GPU parity of the multi-GPU dense path at the configurations bench.py times for N > 1
(BASELINE.json configs[4]: n = 15 at 2 / 4 / 8 GPUs, n = 16 at 8 GPUs).

Every rank is emulated on one GPU, one after the other (independent launches: no kernel
waits on another rank).  Rank h's input is exactly what the equal-split all-to-all
delivers (dist.exchange: block h of every rank's send layout), cut from the full
device-generated matrix.  Each rank's output is checked
  * against the oracle at 4096 seeded coefficients of its own X-mask shard (entries
    regenerated on the host by the independent input module, 1e-12 max|A|),
  * by its own Parseval identity (sum |alpha|^2 over the shard = ||shard||_F^2 / 2^n:
    the shard holds exactly the XOR-diagonals of its X-masks, Theorem 1 per x),
  * at n = 15, bit for bit against the same q-slice of the one-GPU decomposition.
"""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs
from paper_2403_11644_b200 import dist as pdist

pytestmark = pytest.mark.gpu
TOL = 1e-12
SEED = 4


def _torch():
    import torch

    return torch


def _sumsq(t):
    torch = _torch()
    flat = torch.view_as_real(t.reshape(-1))
    tot = 0.0
    for i in range(0, flat.shape[0], 1 << 26):
        c = flat[i:i + (1 << 26)]
        tot += torch.sum(c * c).item()
    return tot


def _recv_block(A, n, world, h):
    """What rank h holds after the all-to-all: recv[g] = A[g R + r][(g ^ h) R + c]."""
    torch = _torch()
    N, R = 1 << n, (1 << n) >> (world.bit_length() - 1)
    V = A.view(world, R, world, R)
    return torch.stack([V[g, :, g ^ h, :] for g in range(world)]).contiguous().view(N, R)


def _shard_qs(n, world, h, count=4096):
    """Seeded global q's whose X-mask lies in rank h's shard (top log2(world) bits of x = h),
    with the shard's edge strings first; returned with their rank-local output indices."""
    rng = np.random.default_rng(7000 + 100 * n + 10 * world + h)
    g = world.bit_length() - 1
    R = (1 << n) >> g
    xs = list(h * R + np.array([0, R - 1, 1, R // 2]))
    zs = [0, (1 << n) - 1, 1 << (n - 1), 1]
    xs += list(h * R + rng.integers(0, R, count - 4))
    zs += list(rng.integers(0, 1 << n, count - 4))
    qs = np.array([ptdr.q_of(int(x), int(z), n) for x, z in zip(xs, zs)], dtype=np.uint64)
    # local index: z_top * 4^(n-g) + (q mod 4^(n-g)) (include/ptdr.h, sharded output)
    w = 2 * (n - g)
    local = (np.array(zs, dtype=np.int64) >> (n - g)) << w | (qs.astype(np.int64) & ((1 << w) - 1))
    return qs, local


@pytest.mark.parametrize("n,world", [(15, 2), (15, 4), (15, 8), (16, 8)])
def test_xshard_bench_configs(gpu, n, world):
    torch = _torch()
    A = ptdr.generate_dense(n, SEED, "general")
    maxabs = max(torch.max(torch.abs(A[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    ref = ptdr.decompose(A) if n == 15 else None
    g = world.bit_length() - 1
    w = 2 * (n - g)
    ws = ptdr.alloc_workspace(n, "general", world, A.device)
    for h in range(world):
        recv = _recv_block(A, n, world, h)
        out = ptdr.decompose_xshard(recv, n, h, world, workspace=ws)
        torch.cuda.synchronize()
        rel = abs(_sumsq(out) - _sumsq(recv) / (1 << n)) / (_sumsq(recv) / (1 << n))
        assert rel < 1e-11, (h, rel)
        del recv
        qs, local = _shard_qs(n, world, h)
        got = out[torch.from_numpy(local).cuda()].cpu().numpy()
        want = oracle.coeffs_generated(n, SEED, 0, qs)
        err = np.max(np.abs(got - want))
        assert err <= TOL * maxabs, (h, err)
        # the global q of every local index (dist.global_q) agrees with the sampled mapping
        for k in (0, 17, len(qs) - 1):
            assert pdist.global_q(h, int(local[k]), n, world) == int(qs[k])
        if ref is not None:
            # rank-local block zt holds the global q range starting at q_of(h, zt, g) << w
            for zt in range(world):
                q0 = ptdr.q_of(h, zt, g) << w
                a = out[zt << w:(zt + 1) << w]
                b = ref[q0:q0 + (1 << w)]
                assert torch.equal(torch.view_as_real(a), torch.view_as_real(b)), (h, zt)
        del out
        torch.cuda.empty_cache()
    del A, ref, ws
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,world,K", [(15, 8, 4), (15, 4, 4), (15, 2, 4), (12, 4, 2), (16, 8, 4)])
def test_subrange_sharded_bench_path(gpu, n, world, K):
    """The overlapped path bench.py runs at N > 1 (dist.decompose_sharded with K
    sub-ranges): rank h's sub-range s is received as the K-sub-range send layout of every
    rank (generate_sendblocks(..., subranges=K), block h of slice s) and decomposed as
    virtual rank h K + s of world K.  Every sub-output equals the matching q-slice of the
    one-GPU decomposition bit for bit (n <= 15), or the oracle at sampled strings (n = 16)."""
    torch = _torch()
    N = 1 << n
    Rp = N // world // K
    gv = (world * K).bit_length() - 1
    w = 2 * (n - gv)
    A = ptdr.generate_dense(n, SEED, "general")
    maxabs = max(torch.max(torch.abs(A[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    ref = ptdr.decompose(A) if n <= 15 else None
    del A
    torch.cuda.empty_cache()
    sends = [ptdr.generate_sendblocks(n, SEED, g, world, subranges=K) for g in range(world)]
    ws = ptdr.alloc_workspace(n, "general", world * K)
    rng = np.random.default_rng(n * 100 + world * 10 + K)
    for h in ([0, world - 1] if n == 16 else range(world)):
        for s in range(K):
            recv = torch.stack([sends[g][s, h] for g in range(world)]).contiguous()
            out = ptdr.decompose_xshard(recv.view(N, Rp), n, h * K + s, world * K, workspace=ws)
            v = h * K + s
            if ref is not None:
                for zt in range(1 << gv):
                    q0 = ptdr.q_of(v, zt, gv) << w
                    assert torch.equal(torch.view_as_real(out[zt << w:(zt + 1) << w]),
                                       torch.view_as_real(ref[q0:q0 + (1 << w)])), (h, s, zt)
            else:
                local = rng.integers(0, out.numel(), 512)
                qs = np.array([pdist.global_q_sub(h, s, int(l), n, world, K) for l in local], dtype=np.uint64)
                got = out[torch.from_numpy(local).cuda()].cpu().numpy()
                want = oracle.coeffs_generated(n, SEED, 0, qs)
                assert np.max(np.abs(got - want)) <= TOL * maxabs, (h, s)
            del recv, out
    del sends, ref
    torch.cuda.empty_cache()


def test_coefficients_xshard_algorithm2(gpu):
    """bench.py's multi-GPU result check: Algorithm 2 (l.302-313) evaluated directly on a
    rank's shard agrees with the oracle, and strings outside the shard give NaN."""
    torch = _torch()
    n, world, h = 13, 8, 5
    A = ptdr.generate_dense(n, SEED, "general")
    recv = _recv_block(A, n, world, h)
    maxabs = torch.max(torch.abs(A)).item()
    del A
    qs, _ = _shard_qs(n, world, h, count=512)
    got = ptdr.coefficients_xshard(recv, n, h, world, qs.astype(np.int64)).cpu().numpy()
    want = oracle.coeffs_generated(n, SEED, 0, qs)
    assert np.max(np.abs(got - want)) <= TOL * maxabs
    other, _ = _shard_qs(n, world, (h + 1) % world, count=8)
    bad = ptdr.coefficients_xshard(recv, n, h, world, other.astype(np.int64)).cpu().numpy()
    assert np.all(np.isnan(bad.real)) and np.all(np.isnan(bad.imag))


@pytest.mark.parametrize("max_ctas", [1, 37, 132])
def test_xshard_grid_cap_is_bitwise_neutral(gpu, max_ctas):
    """ptdr_decompose_xshard_ex_async with a capped persistent grid (SMs left to a concurrent
    all-to-all) gives bit-identical results: tickets are dynamic, the schedule per element is
    not."""
    torch = _torch()
    n, world, h = 14, 2, 1
    A = ptdr.generate_dense(n, SEED, "general")
    recv = _recv_block(A, n, world, h)
    full = ptdr.decompose_xshard(recv, n, h, world)
    capped = ptdr.decompose_xshard(recv, n, h, world, max_ctas=max_ctas)
    assert torch.equal(torch.view_as_real(full), torch.view_as_real(capped))
