"""Physical bf16 expert-parallel dispatch / combine under a placement (config 5).

Per MoE layer on each rank (one process per GPU):
  1. K2/K3 dispatch layout under the placement: pairs ordered by (destination
     group, expert), so each destination rank's rows are one contiguous slice;
  2. mpb_dispatch_gather: hidden-state rows into the send buffer (16-byte
     vectorised, one warp per row);
  3. all-to-all-v over NCCL (torch.distributed.all_to_all_single) with the
     per-rank counts from key_offsets — NCCL 2.2x has no native a2a-v, the
     torch collective lowers to grouped ncclSend/ncclRecv over NVLink;
  4. (expert FFN stand-in: identity) and the reverse all-to-all;
  5. mpb_combine_scatter: weighted fp32 sum of each token's k returned rows,
     in token order (deterministic, no atomics).
The bytes crossing "nodes" (contiguous rank blocks) are what simulate_layer
prices (/root/reference/proj/core/src/simulator.cpp:57-88), here moved for
real; a fused compute+collective kernel over NVLink peer memory is the next
step.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import moeplace as mp
from .distributed import groups_per_rank, send_counts_from_offsets


@dataclass
class A2AStats:
    sent_rows: int = 0
    inter_node_rows: int = 0
    intra_node_rows: int = 0  # includes rows kept on this rank


class ExpertParallelA2A:
    def __init__(self, engine: mp.Engine, placement: mp.Placement, topology: mp.Topology,
                 hidden: int, max_pairs: int, rank: int = 0, world: int = 1, nodes: int = 1,
                 group=None):
        self.eng = engine
        self.dp = engine.placement(placement, topology)
        self.D, self.E = placement.D, placement.E
        self.H = hidden
        self.rank, self.world, self.group = rank, world, group
        self.nodes = nodes
        groups_per_rank(self.D, world)
        dev = engine.device
        self.send = torch.empty(max_pairs, hidden, dtype=torch.bfloat16, device=dev)
        self.back = torch.empty(max_pairs, hidden, dtype=torch.bfloat16, device=dev)
        self.demand = torch.zeros(self.D, self.E, dtype=torch.uint64, device=dev)
        self.sp = torch.empty(max_pairs, dtype=torch.int32, device=dev)
        self.pp = torch.empty(max_pairs, dtype=torch.int32, device=dev)
        self.ko = torch.empty(self.D * self.E + 1, dtype=torch.int64, device=dev)
        per_node = max(1, world // max(1, nodes))
        self.node_of_rank = [r // per_node for r in range(world)]

    def __call__(self, X: torch.Tensor, idx: torch.Tensor, w: torch.Tensor, src: torch.Tensor,
                 stats: A2AStats | None = None) -> torch.Tensor:
        T, k = idx.shape
        n = T * k
        eng = self.eng
        self.demand.zero_()
        eng.dispatch_layout(idx, self.dp, src=src, demand=self.demand,
                            perm_out=(self.sp[:n], self.pp[:n], self.ko))
        eng.dispatch_gather(X, self.sp[:n], k, out=self.send[:n])
        counts = send_counts_from_offsets(self.ko.cpu().numpy(), self.D, self.E, self.world)
        if stats is not None:
            for r, c in enumerate(counts):
                stats.sent_rows += int(c)
                if self.node_of_rank[r] == self.node_of_rank[self.rank]:
                    stats.intra_node_rows += int(c)
                else:
                    stats.inter_node_rows += int(c)
        if self.world == 1:
            back = self.send[:n]  # the all-to-all degenerates to a local permute
        else:
            sc = torch.from_numpy(counts).to(X.device)
            rc = torch.empty_like(sc)
            dist.all_to_all_single(rc, sc, group=self.group)
            rcl = rc.cpu().tolist()
            scl = counts.tolist()
            recv = torch.empty(sum(rcl), self.H, dtype=torch.bfloat16, device=X.device)
            dist.all_to_all_single(recv, self.send[:n], rcl, scl, group=self.group)
            # expert FFN stand-in: identity on the received rows
            back = self.back[:n]
            dist.all_to_all_single(back, recv, scl, rcl, group=self.group)
        return eng.combine_scatter(back, self.pp[:n], w)


def source_groups_cluster(domains: np.ndarray, domain_route, seed: int = 0) -> np.ndarray:
    """Cluster routing: a request of domain d starts on a group of its
    cluster's group set (uniform pick when several)."""
    rng = np.random.default_rng(seed)
    return np.array([g[0] if len(g) == 1 else g[rng.integers(len(g))]
                     for g in (domain_route[int(d)] for d in domains)], np.uint8)
