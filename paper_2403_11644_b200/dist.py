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


def exchange(send: torch.Tensor, group=None, recv: torch.Tensor | None = None) -> torch.Tensor:
    """Equal-split all-to-all of the [world][R][R] send blocks.

    Rank h receives block h of every rank g: recv[g][r][c] = A[g*R + r][(g ^ h)*R + c],
    which read as a [2^n][R] row-major array is A_local[i][c] = A[i][((i >> (n-log2 world)) ^ h)*R + c].
    """
    if recv is None:
        recv = torch.empty_like(send)
    dist.all_to_all_single(recv.view(-1), send.contiguous().view(-1), group=group)
    return recv


def decompose_sharded(send: torch.Tensor, n: int, group=None, out=None, recv=None, workspace=None,
                      stream=None) -> torch.Tensor:
    """All-to-all + per-rank decomposition.  Returns the rank-local coefficients
    (4^n / world, ordering in include/ptdr.h ptdr_decompose_xshard_async)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    recv = exchange(send, group, recv)
    N = 1 << n
    return decompose_xshard(recv.view(N, N // world), n, rank, world, out=out,
                            workspace=workspace, stream=stream)


def global_q(rank: int, local_index: int, n: int, world: int) -> int:
    """Global q of the rank-local output index (host bookkeeping)."""
    g = world.bit_length() - 1
    w = 2 * (n - g)
    zt = local_index >> w
    return (q_of(rank, zt, g) << w) | (local_index & ((1 << w) - 1))


def global_q_array(rank: int, n: int, world: int):
    """Vectorised global_q for all local indices of a rank (numpy int64)."""
    import numpy as np

    g = world.bit_length() - 1
    w = 2 * (n - g)
    local = np.arange((1 << (2 * n)) // world, dtype=np.int64)
    zt = local >> w
    top = np.array([q_of(rank, int(v), g) for v in range(1 << g)], dtype=np.int64)
    return (top[zt] << w) | (local & ((1 << w) - 1))


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
