"""Multi-process host logic of the X-mask sharded path (CPU, gloo, world_size 2 and 4).

The CUDA per-rank computation is tested on the GPU (test_gpu_configs.py emulates every
rank's shard bitwise); here the exchange, the shard layout contract the kernels rely on,
and the rank-local output ordering are checked with real torch.distributed processes.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, result_q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ptdr_inputs
        from paper_2403_11644_b200 import dist as pdist
        from paper_2403_11644_b200 import xz_of

        N = 1 << n
        R = N // world
        g = world.bit_length() - 1
        rows = ptdr_inputs.dense(n, 4, "general", row0=rank * R, nrows=R)
        # send layout [world][R][R]: block b = my rows x column block (rank ^ b)
        send = np.stack([rows[:, (rank ^ b) * R:((rank ^ b) + 1) * R] for b in range(world)])
        assert np.array_equal(send.reshape(-1), pdist.sendblocks_host(rows, n, rank, world).reshape(-1))
        send_t = torch.from_numpy(np.ascontiguousarray(send))
        recv = pdist.exchange(send_t)
        local = recv.numpy().reshape(N, R)
        A = ptdr_inputs.dense(n, 4, "general")
        ok = True
        # shard contract: A_local[i][c] = A[i][((i >> (n-g)) ^ rank) * R + c]
        for i in range(N):
            blk = (i >> (n - g)) ^ rank
            ok &= np.array_equal(local[i], A[i, blk * R:(blk + 1) * R])
        # every XOR-diagonal the rank owns is available locally:
        # v_x[i] = A[i][i ^ x] = A_local[i][(i ^ x) & (R-1)] for x with x >> (n-g) == rank
        for x in range(rank * R, (rank + 1) * R):
            i = np.arange(N)
            ok &= np.array_equal(local[i, (i ^ x) & (R - 1)], A[i, i ^ x])
        # rank-local output order: global q of each local index, all with x_top == rank
        qs = pdist.global_q_array(rank, n, world)
        for q in qs[:: max(1, qs.size // 64)]:
            x, _ = xz_of(int(q), n)
            ok &= (x >> (n - g)) == rank
        result_q.put((rank, bool(ok), qs.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 5), (4, 6)])
def test_xmask_exchange_and_layout(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allq = []
    for rank, ok, qs in sorted(results):
        assert ok, f"rank {rank} layout/contract check failed"
        allq += qs
    # the ranks' outputs tile the global q range exactly once
    assert sorted(allq) == list(range(4 ** n))


def _band_worker(rank, world, port, n, structure, result_q):
    """z-sharded structured path: every rank holds the whole band, computes its z-slice of
    every block (here with the oracle, standing in for the kernels), and the gloo all_gather
    + reorder of dist.gather_band_sharded must rebuild the one-GPU output layout."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import ptdr_inputs
        from paper_2403_11644_b200 import dist as pdist
        from paper_2403_11644_b200 import q_of

        N = 1 << n
        blocks = n + 1 if structure == "tridiagonal" else 1
        gidx = pdist.zshard_index(rank, n, world, blocks)       # global index of each local one
        b, z = gidx >> n, gidx & (N - 1)
        xs = (1 << b) - 1 if structure == "tridiagonal" else np.zeros_like(b)
        qs = np.array([q_of(int(x), int(zz), n) for x, zz in zip(xs, z)], dtype=np.uint64)
        if structure == "tridiagonal":
            sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
            local = oracle.coeffs_tridiagonal(sub, main, sup, qs)
        else:
            d = ptdr_inputs.band(n, 3, "diagonal")
            local = oracle.coeffs_diagonal(d, qs)
        full = pdist.gather_band_sharded(torch.from_numpy(np.ascontiguousarray(local)), n, blocks)
        result_q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,structure", [(2, 5, "tridiagonal"), (4, 6, "tridiagonal"),
                                               (2, 6, "diagonal")])
def test_band_zshard_gather(world, n, structure):
    import oracle
    import ptdr_inputs
    from paper_2403_11644_b200 import dist as pdist
    from paper_2403_11644_b200 import q_of

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, n, structure, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N = 1 << n
    blocks = n + 1 if structure == "tridiagonal" else 1
    xs = [(1 << b) - 1 for b in range(blocks)] if structure == "tridiagonal" else [0]
    qs = np.array([q_of(x, z, n) for x in xs for z in range(N)], dtype=np.uint64)
    if structure == "tridiagonal":
        sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
        want = oracle.coeffs_tridiagonal(sub, main, sup, qs)
    else:
        want = oracle.coeffs_diagonal(ptdr_inputs.band(n, 3, "diagonal"), qs)
    for rank, full in results:
        assert np.array_equal(full, want), f"rank {rank}"
    # the host-side assembly agrees with the collective one, and the slices tile the output
    parts = [want[pdist.zshard_index(r, n, world, blocks)] for r in range(world)]
    assert np.array_equal(pdist.assemble_zshards(parts, n, blocks), want)
    allidx = np.concatenate([pdist.zshard_index(r, n, world, blocks) for r in range(world)])
    assert np.array_equal(np.sort(allidx), np.arange(blocks << n))


def _peer_blob_worker(rank, world, port, result_q):
    """Host logic of the peer-pull setup: the (handle, offset) blobs gathered over a real
    process group come back in rank order and map to base + offset (fake handles, no GPU)."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_11644_b200 import dist as pdist

        mine = (bytes([rank]) * 64, 4096 * rank + 16)
        blobs = pdist._exchange_objects(mine)
        bases = {}

        def fake_open(handle):
            r = handle[0]
            bases[r] = 0x7000_0000_0000 + (r << 32)
            return bases[r]

        ptrs, opened = pdist.peer_pointers(blobs, rank, 0xDEAD0000, fake_open)
        result_q.put((rank, ptrs, sorted(bases)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_handle_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_blob_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ptrs, opened in res:
        assert len(ptrs) == world
        assert opened == [r for r in range(world) if r != rank]       # never maps itself
        for r, pt in enumerate(ptrs):
            want = 0xDEAD0000 if r == rank else 0x7000_0000_0000 + (r << 32) + 4096 * r + 16
            assert pt == want


def _subrange_worker(rank, world, port, n, K, result_q):
    """Sub-range overlapped exchange (dist.exchange_async): every one of the K equal-split
    all-to-alls must deliver exactly the A_local of virtual rank rank*K + s of world*K (the
    input contract of ptdr_decompose_xshard_async), so the K decompositions can start one
    by one as their sub-range lands."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ptdr_inputs
        from paper_2403_11644_b200 import dist as pdist
        from paper_2403_11644_b200 import xz_of

        N = 1 << n
        R = N // world
        Rp = R // K
        gv = (world * K).bit_length() - 1
        rows = ptdr_inputs.dense(n, 4, "general", row0=rank * R, nrows=R)
        send = torch.from_numpy(np.ascontiguousarray(pdist.sendblocks_host(rows, n, rank, world, K)))
        recv, works = pdist.exchange_async(send)
        A = ptdr_inputs.dense(n, 4, "general")
        ok = True
        allq = []
        for s in range(K):
            works[s].wait()
            local = recv[s].numpy().reshape(N, Rp)
            v = rank * K + s
            for i in range(N):
                blk = (i >> (n - gv)) ^ v
                ok &= np.array_equal(local[i], A[i, blk * Rp:(blk + 1) * Rp])
            # sub-output s covers exactly the X-masks of virtual rank v
            for li in range(0, (1 << (2 * n)) // (world * K), 7):
                q = pdist.global_q_sub(rank, s, li, n, world, K)
                x, _ = xz_of(q, n)
                ok &= (x >> (n - gv)) == v
                allq.append(q)
        result_q.put((rank, bool(ok), allq))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,K", [(2, 6, 2), (2, 6, 4), (4, 7, 2)])
def test_subrange_exchange_contract(world, n, K):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_subrange_worker, args=(r, world, port, n, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allq = []
    for rank, ok, qs in sorted(results):
        assert ok, f"rank {rank}: sub-range exchange contract failed"
        allq += qs
    assert len(set(allq)) == len(allq)
