"""Warm per-kernel GPU timings (CUDA events, launches pre-queued) at the DSv3 step shape."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402

T, E, k, D, L, P = 65536, 256, 8, 8, 58, 1022
ONCE = "--once" in sys.argv  # each case launched once, untimed (for ncu captures)
argv = [a for a in sys.argv[1:] if a != "--once"]
SMS = int(argv[0]) if argv else 0  # SM budget (the side context's, e.g. 20)
CONFINE = len(argv) > 1 and argv[1] == "confined"  # run inside an SM partition
if CONFINE:
    part = mp.SmPartition(0, SMS)
    torch.cuda.set_stream(part.side)
    eng = mp.Engine(0, stream=part.side)
    eng.set_sm_partition(part.side_sms)
    print(f"confined to a {part.side_sms}-SM partition")
else:
    eng = mp.Engine(0)
    if SMS:
        eng.set_sm_budget(SMS)
rng = np.random.default_rng(0)
idx = torch.from_numpy(np.argsort(rng.random((T, E), dtype=np.float32), axis=1)[:, :k]
                       .astype(np.int32)).cuda()
src = torch.from_numpy((np.arange(T) // 16 % D).astype(np.uint8)).cuda()
dom = torch.from_numpy((np.arange(T) // 16 % 8).astype(np.uint16)).cuda()
top = mp.Topology.contiguous(D, 1, D, 1, 2)
pl = mp.Placement([list(range(d * 32, d * 32 + 32)) for d in range(D)], E, 0, 32)
dp = eng.placement(pl, top)
demand = torch.zeros(D, E, dtype=torch.uint64, device="cuda")
demand2 = torch.zeros(D, E, dtype=torch.uint64, device="cuda")
src2 = torch.from_numpy((np.arange(T) // 16 * 3 % D).astype(np.uint8)).cuda()
pop = torch.zeros(8, E, dtype=torch.uint64, device="cuda")
sp = torch.empty(T * k, dtype=torch.int32, device="cuda")
pp = torch.empty(T * k, dtype=torch.int32, device="cuda")
ko = torch.empty(D * E + 1, dtype=torch.int64, device="cuda")
co = torch.zeros(E, E, dtype=torch.uint64, device="cuda")
dem_l = torch.randint(0, 100, (L, D, E), device="cuda").to(torch.uint64)
luts = torch.from_numpy(np.stack([mp.host_dest_lut(pl, top.group_to_node)] * P)).cuda()
g2n = torch.tensor(top.group_to_node, dtype=torch.uint8, device="cuda")
out = (torch.zeros(P, L, dtype=torch.uint64, device="cuda"),
       torch.zeros(P, L, dtype=torch.uint64, device="cuda"),
       torch.zeros(P, L, D, dtype=torch.uint64, device="cuda"))
fin = (torch.empty(P * L, 6, dtype=torch.float64, device="cuda"),
       torch.empty(P * L, D, dtype=torch.float64, device="cuda"))
cost = mp.CostModelParams(7168, 2)

cases = {
    "layout+perm+tag": lambda: eng.dispatch_layout(idx, dp, src=src, tag=dom, n_tags=8,
                                                   demand=demand, tag_pop=pop,
                                                   perm_out=(sp, pp, ko)),
    "layout+perm+tag+src2": lambda: eng.dispatch_layout(idx, dp, src=src, tag=dom, n_tags=8,
                                                        demand=demand, tag_pop=pop,
                                                        perm_out=(sp, pp, ko), src2=src2,
                                                        demand2=demand2),
    "layout demand-only": lambda: eng.dispatch_layout(idx, dp, src=src, permutation=False,
                                                      demand=demand),
    "coactivation": lambda: eng.coactivation(idx, E, out=co),
    "score P=1022 x L=58": lambda: eng.score_placements(dem_l, luts, g2n, D, row_node=g2n,
                                                        out=out),
    "finalize 59K cells": lambda: eng.finalize(out[0].view(-1), out[1].view(-1),
                                               out[2].view(-1, D), D, cost, top, out=fin[0],
                                               payload=fin[1]),
}
if ONCE:
    for name, fn in cases.items():
        fn()
        torch.cuda.synchronize()
        print(f"{name}: launched once")
    eng.sync()
    sys.exit(0)
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n0 = eng.launches
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # keep the GPU busy while the host queues the 20 calls, so the events time
    # the kernels, not the host's launch rate
    torch.cuda._sleep(int(2e7))
    s.record()
    for _ in range(20):
        fn()
    e.record()
    torch.cuda.synchronize()
    print(f"{name:24s} {s.elapsed_time(e) / 20 * 1e3:9.2f} us  ({(eng.launches - n0) // 20} launches)")
eng.sync()
