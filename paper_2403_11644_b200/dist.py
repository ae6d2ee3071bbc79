"""Multi-GPU paths.

Dense GENERAL: X-mask sharding.

One process per GPU.  Rank g starts with its row block of A in the
column-block-major send layout send[b][r][c] = A[g*R + r][(g ^ b)*R + c]
(ptdr_generate_sendblocks_async writes it directly), one equal-split
all-to-all over NCCL turns row blocks into X-mask shards, and every rank then
gathers and transforms its own XOR-diagonals with no further communication
(ptdr_decompose_xshard_async).  The exchange is the only collective on the path.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import decompose_xshard, decompose_zshard, q_of


def _nvtx(name):
    """NVTX range (for nsys timelines of the exchange / kernel overlap); no-op without CUDA."""
    import contextlib

    if torch.cuda.is_available():
        return torch.cuda.nvtx.range(name)
    return contextlib.nullcontext()


def exchange(send: torch.Tensor, group=None, recv: torch.Tensor | None = None) -> torch.Tensor:
    """Equal-split all-to-all of the send blocks (one sub-range: send is [world][R*R] or
    [1][world][R*R]).

    Rank h receives block h of every rank g: recv[g][r][c] = A[g*R + r][(g ^ h)*R + c],
    which read as a [2^n][R] row-major array is A_local[i][c] = A[i][((i >> (n-log2 world)) ^ h)*R + c].
    """
    if recv is None:
        recv = torch.empty_like(send)
    with _nvtx("ptdr.exchange"):
        dist.all_to_all_single(recv.view(-1), send.contiguous().view(-1), group=group)
    return recv


def exchange_async(send: torch.Tensor, group=None, recv: torch.Tensor | None = None):
    """Issue the K sub-range all-to-alls of a [K][world][R*R/K] send layout at once
    (async_op=True); returns (recv, works).  works[s].wait() orders sub-range s."""
    if send.dim() == 2:
        send = send.unsqueeze(0)
    if recv is None:
        recv = torch.empty_like(send)
    with _nvtx("ptdr.exchange.issue"):
        works = [dist.all_to_all_single(recv[s].view(-1), send[s].contiguous().view(-1), group=group,
                                        async_op=True) for s in range(send.shape[0])]
    return recv, works


# SMs the decomposition of a sub-range leaves to the next sub-range's all-to-all (NCCL's
# kernels need SMs too; the persistent pipeline otherwise takes every SM and the exchange
# would only start after it).  The last sub-range, with nothing left in flight, takes all.
COMM_SMS = 16


def decompose_sharded(send: torch.Tensor, n: int, group=None, out=None, recv=None, workspace=None,
                      stream=None, comm_sms: int = COMM_SMS) -> torch.Tensor:
    """All-to-all + per-rank decomposition, overlapped by sub-range.

    send: the [K][world][R*R/K] layout of generate_sendblocks(..., subranges=K).  Sub-range
    s of every rank's X-masks is one equal-split all-to-all; all K are issued up front
    (asynchronous on NCCL's stream) and the decomposition of sub-range s -- which is
    ptdr_decompose_xshard_async for virtual rank h K + s of world K -- starts as soon as
    its exchange has landed, while the exchanges of the later sub-ranges are in flight.
    Returns [K][4^n / (world K)]: sub-output s in the layout of virtual rank h K + s
    (global_q_sub).  K = 1 is the plain exchange-then-decompose path.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if send.dim() == 2:
        send = send.unsqueeze(0)
    K = send.shape[0]
    if recv is None:
        recv = torch.empty_like(send)
    N = 1 << n
    Rk = N // world // K
    if out is None:
        out = torch.empty((K, (1 << (2 * n)) // (world * K)), dtype=torch.complex128, device=send.device)
    cur = torch.cuda.current_stream(send.device) if send.is_cuda else None
    recv, works = exchange_async(send, group, recv)
    for s in range(K):
        with _nvtx(f"ptdr.exchange.wait[{s}]"):
            works[s].wait()          # NCCL: the current stream waits for exchange s
        if stream is not None and cur is not None:
            # all_to_all_single is ordered on the current stream only: make `stream` wait
            # for the exchange before the kernels read `recv`
            stream.wait_stream(cur)
        cap = 0
        if world > 1 and s + 1 < K and comm_sms > 0 and send.is_cuda:
            cap = max(1, torch.cuda.get_device_properties(send.device).multi_processor_count - comm_sms)
        with _nvtx(f"ptdr.decompose_xshard[{s}]"):
            decompose_xshard(recv[s].view(N, Rk), n, rank * K + s, world * K, out=out[s],
                             workspace=workspace, stream=stream, max_ctas=cap)
    return out


def global_q(rank: int, local_index: int, n: int, world: int) -> int:
    """Global q of the rank-local output index (host bookkeeping)."""
    g = world.bit_length() - 1
    w = 2 * (n - g)
    zt = local_index >> w
    return (q_of(rank, zt, g) << w) | (local_index & ((1 << w) - 1))


def global_q_sub(rank: int, s: int, local_index: int, n: int, world: int, subranges: int) -> int:
    """Global q of element `local_index` of sub-output s of decompose_sharded (virtual rank
    rank * K + s of world * K)."""
    return global_q(rank * subranges + s, local_index, n, world * subranges)


def global_q_array(rank: int, n: int, world: int):
    """Vectorised global_q for all local indices of a rank (numpy int64)."""
    import numpy as np

    g = world.bit_length() - 1
    w = 2 * (n - g)
    local = np.arange((1 << (2 * n)) // world, dtype=np.int64)
    zt = local >> w
    top = np.array([q_of(rank, int(v), g) for v in range(1 << g)], dtype=np.int64)
    return (top[zt] << w) | (local & ((1 << w) - 1))


def sendblocks_host(rows, n: int, rank: int, world: int, subranges: int = 1):
    """Host (numpy) copy of the send layout of ptdr_generate_sendblocks_async for a rank's
    row block `rows` ([R][2^n]), for tests of the exchange plumbing without a GPU:
    element (s, h, t, r', c') = A[(rank K + t) R' + r'][((rank ^ h) K + (t ^ s)) R' + c']."""
    import numpy as np

    N = 1 << n
    K = subranges
    R = N // world
    Rp = R // K
    out = np.empty((K, world, K, Rp, Rp), dtype=rows.dtype)
    for s in range(K):
        for h in range(world):
            for t in range(K):
                c0 = ((rank ^ h) * K + (t ^ s)) * Rp
                out[s, h, t] = rows[t * Rp:(t + 1) * Rp, c0:c0 + Rp]
    return out.reshape(K, world, K * Rp * Rp)


# ---- structured (DIAGONAL / TRIDIAGONAL): replicated band, z-sharded output -------------
def decompose_band_sharded(band: torch.Tensor, structure, group=None, out=None, workspace=None,
                           stream=None) -> torch.Tensor:
    """Every rank holds the whole band (generated locally from the shared seed: no
    communication) and computes its z-slice of every output block."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    return decompose_zshard(band, structure, rank, world, out=out, workspace=workspace, stream=stream)


def zshard_index(rank: int, n: int, world: int, blocks: int):
    """Global output index of every rank-local element of a z-sharded band output
    (block-major, 2^n/world per block): local b*NL + zl -> global b*2^n + rank*NL + zl."""
    import numpy as np

    NL = (1 << n) // world
    local = np.arange(blocks * NL, dtype=np.int64)
    return (local // NL) * (1 << n) + rank * NL + (local % NL)


def assemble_zshards(parts, n: int, blocks: int):
    """Host-side assembly of the per-rank slices into the one-GPU output layout."""
    import numpy as np

    world = len(parts)
    out = np.empty(blocks << n, dtype=np.asarray(parts[0]).dtype)
    for r, p in enumerate(parts):
        out[zshard_index(r, n, world, blocks)] = np.asarray(p)
    return out


def gather_band_sharded(local: torch.Tensor, n: int, blocks: int, group=None) -> torch.Tensor:
    """all_gather the slices and reorder them into the one-GPU output (for users who need
    the whole result on every rank; not part of the timed path)."""
    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    NL = (1 << n) // world
    stacked = torch.stack([p.view(blocks, NL) for p in parts], dim=1)  # [blocks][world][NL]
    return stacked.reshape(blocks << n)


# ---- dense, fused exchange: peer pull over NVLink -----------------------
def _exchange_objects(obj, group=None):
    world = dist.get_world_size(group)
    objs = [None] * world
    dist.all_gather_object(objs, obj, group=group)
    return objs


def peer_pointers(blobs, rank: int, local_ptr: int, open_fn):
    """Device addresses of every rank's shard from the gathered (handle, offset) blobs: the
    local shard as is, peers mapped through `open_fn(handle) -> base` plus their offset.
    Returns (pointers in rank order, bases to close)."""
    ptrs, opened = [], []
    for r, (handle, offset) in enumerate(blobs):
        if r == rank:
            ptrs.append(int(local_ptr))
        else:
            base = open_fn(handle)
            opened.append(base)
            ptrs.append(base + int(offset))
    return ptrs, opened


def open_peer_shards(shard: torch.Tensor, group=None):
    """CUDA IPC exchange of the ranks' row-block shards.  Returns (device pointers of all
    shards in rank order, close()).  Collective over `group`."""
    from . import ipc_close, ipc_handle, ipc_open

    rank = dist.get_rank(group)
    blobs = _exchange_objects(ipc_handle(shard), group)
    ptrs, opened = peer_pointers(blobs, rank, shard.data_ptr(), ipc_open)

    def close():
        for b in opened:
            ipc_close(b)

    return ptrs, close


def decompose_peer_sharded(shard: torch.Tensor, n: int, ptrs, group=None, out=None, workspace=None,
                           stream=None) -> torch.Tensor:
    """Fused exchange + decomposition: rank h's phase-A tiles read the rows they need
    directly from the owning rank's shard (TMA over NVLink), no all-to-all, no receive
    buffer.  Every shard must be complete before the call (barrier) and stay unmodified
    until every rank has finished (the caller's barrier after synchronising)."""
    from . import decompose_peer

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    return decompose_peer(ptrs, n, rank, world, out=out, workspace=workspace, stream=stream,
                          device=shard.device)
