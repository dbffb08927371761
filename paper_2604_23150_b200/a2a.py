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
real.

`enable_p2p()` replaces 2-5 with the fused NVLink path (K6-P2P): receive
buffers are symmetric memory mapped into every rank; one kernel gathers each
sorted pair's row straight into the destination rank's buffer (remote stores).
The return leg is pulled by default: the combine reads each token's k rows
out of the peers' buffers inside the weighted sum (remote loads);
`combine="push"` instead writes the received rows back into their source
ranks' symmetric `back` buffers at the sources' sorted positions and the
source combines from local memory (measured slower: profiles/r01_a2a_n*.json). No send staging, no NCCL payload collective; the
per-destination counts travel through peer memory too. Cross-rank ordering
uses the symmetric-memory barrier (stream-ordered signal pads).
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
        self.p2p = False
        self.phase_events = None  # list -> per-step (start, counts, dispatch, combine) events

    def enable_p2p(self, capacity_rows: int, combine: str = "pull", dispatch: str = "push",
                   max_tokens: int | None = None) -> None:
        """Maps a `capacity_rows` x H bf16 receive buffer and a [world][world]
        count matrix of every rank into this process (symmetric memory).
        dispatch="pull": each rank also stages its hidden states (up to
        `max_tokens` rows), sorted pairs and key offsets in symmetric memory,
        and destinations copy their rows out of the sources' buffers
        (mpb_dispatch_pull); "push": sources store rows into the destinations'
        buffers (mpb_dispatch_p2p). Same receive buffer either way."""
        dev = self.eng.device
        self.dispatch_mode = dispatch
        if max_tokens is None:
            max_tokens = self.send.shape[0]
        if self.world == 1:
            self.recv = torch.empty(capacity_rows, self.H, dtype=torch.bfloat16, device=dev)
            self.back_sym = self.back
            self.peer_back = torch.tensor([self.back.data_ptr()], dtype=torch.uint64, device=dev)
            self.cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            self.peer_recv = torch.tensor([self.recv.data_ptr()], dtype=torch.uint64, device=dev)
            self.peer_cnt = torch.tensor([self.cnt.data_ptr()], dtype=torch.uint64, device=dev)
            self.hdl = None
            if dispatch == "pull":
                self.x_sym = torch.empty(max_tokens, self.H, dtype=torch.bfloat16, device=dev)
                self.peer_x = torch.tensor([self.x_sym.data_ptr()], dtype=torch.uint64, device=dev)
                self.peer_sp = torch.tensor([self.sp.data_ptr()], dtype=torch.uint64, device=dev)
                self.peer_ko = torch.tensor([self.ko.data_ptr()], dtype=torch.uint64, device=dev)
        else:
            import torch.distributed._symmetric_memory as symm_mem
            gname = (self.group or dist.group.WORLD).group_name
            cap = torch.tensor([capacity_rows], dtype=torch.int64, device=dev)
            dist.all_reduce(cap, op=dist.ReduceOp.MAX, group=self.group)  # same size everywhere
            capacity_rows = int(cap.item())
            self.recv = symm_mem.empty(capacity_rows, self.H, dtype=torch.bfloat16, device=dev)
            self.hdl = symm_mem.rendezvous(self.recv, gname)
            mx = torch.tensor([self.send.shape[0]], dtype=torch.int64, device=dev)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self.group)
            self.back_sym = symm_mem.empty(int(mx.item()), self.H, dtype=torch.bfloat16,
                                           device=dev)
            hb = symm_mem.rendezvous(self.back_sym, gname)
            self.peer_back = torch.tensor(list(hb.buffer_ptrs), dtype=torch.uint64, device=dev)
            self._hb = hb
            self.cnt = symm_mem.empty(self.world * self.world, dtype=torch.int64, device=dev)
            hc = symm_mem.rendezvous(self.cnt, gname)
            self.peer_recv = torch.tensor(list(self.hdl.buffer_ptrs), dtype=torch.uint64,
                                          device=dev)
            self.peer_cnt = torch.tensor(list(hc.buffer_ptrs), dtype=torch.uint64, device=dev)
            self._hc = hc
            if dispatch == "pull":
                mt = torch.tensor([max_tokens], dtype=torch.int64, device=dev)
                dist.all_reduce(mt, op=dist.ReduceOp.MAX, group=self.group)
                self.x_sym = symm_mem.empty(int(mt.item()), self.H, dtype=torch.bfloat16,
                                            device=dev)
                hx = symm_mem.rendezvous(self.x_sym, gname)
                # the layout writes the sorted pairs / key offsets straight into
                # symmetric buffers the destinations read
                sp = symm_mem.empty(int(mx.item()), dtype=torch.int32, device=dev)
                hs = symm_mem.rendezvous(sp, gname)
                ko = symm_mem.empty(self.D * self.E + 1, dtype=torch.int64, device=dev)
                hk = symm_mem.rendezvous(ko, gname)
                self.sp, self.ko = sp, ko
                self.peer_x = torch.tensor(list(hx.buffer_ptrs), dtype=torch.uint64, device=dev)
                self.peer_sp = torch.tensor(list(hs.buffer_ptrs), dtype=torch.uint64, device=dev)
                self.peer_ko = torch.tensor(list(hk.buffer_ptrs), dtype=torch.uint64, device=dev)
                self._hx, self._hs, self._hk = hx, hs, hk
        self.capacity = capacity_rows
        self.combine_mode = combine  # "pull": remote loads in the combine (default); "push"
        self.p2p = True

    def _barrier(self):
        if self.hdl is not None:
            self.hdl.barrier(channel=0)

    def __call__(self, X: torch.Tensor, idx: torch.Tensor, w: torch.Tensor, src: torch.Tensor,
                 stats: A2AStats | None = None) -> torch.Tensor:
        T, k = idx.shape
        n = T * k
        eng = self.eng
        self.demand.zero_()
        eng.dispatch_layout(idx, self.dp, src=src, demand=self.demand,
                            perm_out=(self.sp[:n], self.pp[:n], self.ko))
        if self.p2p:
            return self._p2p(X, idx, w, n, k, stats)
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

    def _count_stats(self, stats: A2AStats) -> None:
        counts = send_counts_from_offsets(self.ko.cpu().numpy(), self.D, self.E, self.world)
        for r, c in enumerate(counts):
            stats.sent_rows += int(c)
            if self.node_of_rank[r] == self.node_of_rank[self.rank]:
                stats.intra_node_rows += int(c)
            else:
                stats.inter_node_rows += int(c)

    def _p2p(self, X, idx, w, n, k, stats):
        # the symmetric-memory barrier and the x_sym staging copy are issued on
        # torch's current stream; run them on the engine's stream so the
        # barrier orders the P2P kernels (which the engine launches there)
        with torch.cuda.stream(self.eng.stream):
            return self._p2p_body(X, idx, w, n, k, stats)

    def _p2p_body(self, X, idx, w, n, k, stats):
        eng = self.eng
        span = groups_per_rank(self.D, self.world) * self.E
        if stats is not None:
            self._count_stats(stats)
        ph = self.phase_events  # optional per-phase device timing (tools/bench_a2a.py)
        if ph is not None:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ph.append(ev)
            ev[0].record(eng.stream)
        pull = self.dispatch_mode == "pull"
        if pull:  # stage the hidden states where the destinations can read them
            self.x_sym[:X.shape[0]].copy_(X)
        eng.a2a_put_counts(self.ko, span, self.world, self.rank, self.peer_cnt)
        self._barrier()  # every rank's counts (and staged rows / pairs) are visible
        if ph is not None:
            ev[1].record(eng.stream)
        if pull:
            eng.dispatch_pull(self.cnt, self.peer_x, self.peer_sp, self.peer_ko, k, self.H, span,
                              self.world, self.rank, self.recv, self.capacity)
        else:
            eng.dispatch_p2p(X, self.sp[:n], k, self.cnt, self.ko, span, self.world, self.rank,
                             self.peer_recv, self.capacity)
        self._barrier()  # every row has landed in its destination buffer
        if ph is not None:
            ev[2].record(eng.stream)
        # expert FFN stand-in: identity on this rank's received rows
        if self.combine_mode == "push":
            # each rank pushes the rows it received (after its experts) back to
            # their source ranks' `back` buffers, in the sources' sorted order
            eng.return_p2p(self.recv, self.capacity, self.cnt, self.world, self.rank,
                           self.peer_back)
            self._barrier()  # every row is home
            Y = eng.combine_scatter(self.back_sym[:n], self.pp[:n], w)
            if ph is not None:
                ev[3].record(eng.stream)
            return Y
        self._barrier()  # every rank's experts are done with its rows
        Y = torch.empty(idx.shape[0], self.H, dtype=torch.bfloat16, device=X.device)
        eng.combine_p2p(self.pp[:n], w, self.H, self.cnt, self.ko, span, self.world, self.rank,
                        self.peer_recv, Y)
        self._barrier()  # peers have read their rows back: buffers reusable
        if ph is not None:
            ev[3].record(eng.stream)
        return Y


def source_groups_cluster(domains: np.ndarray, domain_route, seed: int = 0) -> np.ndarray:
    """Cluster routing: a request of domain d starts on a group of its
    cluster's group set (uniform pick when several)."""
    rng = np.random.default_rng(seed)
    return np.array([g[0] if len(g) == 1 else g[rng.integers(len(g))]
                     for g in (domain_route[int(d)] for d in domains)], np.uint8)
