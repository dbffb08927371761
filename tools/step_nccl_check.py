#!/usr/bin/env python
"""Multi-rank check of the C++ step's own NCCL collectives (torchrun):
the same routed step with the collectives issued by the plan (per-chunk
all-reduce of the demand beside the routers, tag / co-activation all-reduce,
all-gather of the sharded score rows, captured into the CUDA graph) and with
torch.distributed collectives between the two phases (MPB_STEP_NCCL=0) give
bit-identical statistics and LayerSim tables on every rank. Rank 0 prints one
JSON line; exit 1 on mismatch."""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, WorkloadSpec  # noqa: E402


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["MPB_ROUTER_NO_SPLIT"] = "1"
    spec = WorkloadSpec("tiny", 6, 8192, 512, 64, 8, 1, True, groups=8, nodes=2, domains=4,
                        preferred=8, candidates=64)
    out = {}
    for mode in ("1", "0"):
        os.environ["MPB_STEP_NCCL"] = mode
        eng = mp.Engine(local)
        pipe = RoutingPipeline(spec, eng, rank, world, resident=True)
        if mode == "1":
            pipe.capture()  # the graphed step carries the NCCL collectives
        for _ in range(2):
            pipe.step()
        torch.cuda.synchronize()
        out[mode] = [pipe.stats.clone(), pipe.fin_cl[0].clone(), pipe.fin_cl[1].clone(),
                     pipe.fin_rr[0].clone()]
        del pipe
    same = all(torch.equal(a, b) for a, b in zip(out["1"], out["0"]))
    flag = torch.tensor([int(same)], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    ok = bool(flag.item())
    if rank == 0:
        print(json.dumps({"check": "step_nccl_in_plan_vs_torch", "world": world,
                          "all_ranks_bit_identical": ok}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
