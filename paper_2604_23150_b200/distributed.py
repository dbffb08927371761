"""Multi-GPU plumbing for the routed step: one process per GPU over
torch.distributed (NCCL on the B200s, gloo in CPU tests).

* EP groups are dealt contiguously over ranks (D % world == 0): rank r hosts
  groups [r·D/world, (r+1)·D/world). "Nodes" are contiguous rank blocks
  (GPU groups standing in for nodes), matching
  Topology::contiguous (/root/reference/proj/core/src/placement.cpp:75-94).
* The only collective of the statistics path is one all-reduce(sum) of the
  fused uint64 statistics buffer (integer sums: bit-exact in any order).
* Candidate scoring is sharded: rank r prices candidates [r·P/world,
  (r+1)·P/world) of the global demand and the LayerSim rows are all-gathered
  (SURVEY §8e collective 2); every rank ends with the full table.
* The bf16 dispatch / combine all-to-all-v uses the K3 permutation's
  key_offsets to size the per-rank sends (a2a.py).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def groups_per_rank(D: int, world: int) -> int:
    if world < 1 or D % world != 0:
        raise ValueError(f"EP groups D={D} must be a multiple of world={world}")
    return D // world


def rank_of_group(g: int, D: int, world: int) -> int:
    return g // groups_per_rank(D, world)


def node_of_rank(r: int, world: int, nodes: int) -> int:
    if world % nodes != 0 and nodes <= world:
        raise ValueError("nodes must divide world")
    return r // max(1, world // nodes) if nodes <= world else r


def send_counts_from_offsets(key_offsets: np.ndarray, D: int, E: int, world: int) -> np.ndarray:
    """Pairs this rank sends to each destination rank: the permutation is
    ordered by (dest group, expert), groups are contiguous per rank, so rank
    r's slice is [key_offsets[first_group(r)*E], key_offsets[first_group(r+1)*E])."""
    gpr = groups_per_rank(D, world)
    bounds = [int(key_offsets[r * gpr * E]) for r in range(world)] + [int(key_offsets[D * E])]
    return np.diff(np.asarray(bounds, np.int64))


def all_reduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Sums a uint64 statistics buffer across ranks (viewed as int64: two's
    complement addition is the same bit pattern)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats.view(torch.int64), op=dist.ReduceOp.SUM, group=group)
    return stats


def exchange_counts(send_counts: torch.Tensor, group=None) -> torch.Tensor:
    """all-to-all of the per-destination pair counts (one int64 per rank)."""
    recv = torch.empty_like(send_counts)
    dist.all_to_all_single(recv, send_counts, group=group)
    return recv


def shard_bounds(P: int, world: int, rank: int):
    """Candidate slice of `rank` when P splits evenly over the ranks, else
    None (every rank scores all P)."""
    if world <= 1 or P % world != 0:
        return None
    per = P // world
    return rank * per, (rank + 1) * per


def gather_shards(full: torch.Tensor, rows_per_rank: int, group=None) -> torch.Tensor:
    """All-gathers `full` in place along dim 0: rank r owns rows
    [r·rows_per_rank, (r+1)·rows_per_rank) on entry, every rank holds all of
    them on return (bit copies: float64 LayerSims stay bit-identical)."""
    world = dist.get_world_size(group)
    chunks = list(full.split(rows_per_rank, dim=0))
    if len(chunks) != world:
        raise ValueError("gather_shards: rows do not split evenly over the ranks")
    mine = chunks[dist.get_rank(group)].clone()
    dist.all_gather(chunks, mine, group=group)
    return full
