"""Where the DSv3 step's non-router time goes (experiments).
  python tools/step_probe.py [variant ...]
    full / nocoact / noscore : the graphed step timed with parts of the side
        stream's statistics work switched off (those variants do not produce
        the step's full results)
    timeline : one eager step with MPB_STEP_PROBE=1 — per chunk, when its
        router finished (main stream) and when its statistics tails + pricing
        finished (side stream; the last chunk's on main), in ms from the start"""
import ctypes as C
import gc
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import _abi, moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

eng = mp.Engine(0)
for v in sys.argv[1:] or ["full", "nocoact", "noscore"]:
    over = {"coact": False} if v == "nocoact" else {}
    os.environ["MPB_SCORE_PER_CHUNK"] = "0" if v == "noscore" else "1"
    os.environ["MPB_STEP_PROBE"] = "1" if v == "timeline" else "0"
    spec = spec_for("dsv3", **over)
    pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
    for _ in range(2):
        pipe.step()
    torch.cuda.synchronize()
    if v == "timeline":
        for _ in range(3):
            pipe.step()
        torch.cuda.synchronize()
        n = 64
        buf = (C.c_float * n)()
        got = _abi.lib().mpb_debug_step_probe(pipe.plan.handle, buf, C.c_size_t(n))
        nc = (got - 1) // 2
        chunks = [pipe.plan_chunks[c] for c in range(nc)] if hasattr(pipe, "plan_chunks") else [None] * nc
        print(f"timeline (eager, ms from start): step end {buf[2 * nc]:.3f}")
        for c in range(nc):
            print(f"  chunk {c}: router done {buf[c]:7.3f}  tails+pricing done {buf[nc + c]:7.3f}  "
                  f"lag {buf[nc + c] - buf[c]:6.3f}", flush=True)
    else:
        ok = pipe.capture()
        for _ in range(2):
            pipe.step()
        torch.cuda.synchronize()
        pipe.plan.timing_reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        for _ in range(5):
            pipe.step(timed_router=True)
        b.record(eng.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        r = sum(pipe.graph_router_ms()) / len(pipe.graph_router_ms()) if ok else float("nan")
        print(f"{v:8s} graph={ok} step {ms:.3f} ms; router {r:.4f} ms/layer x {spec.layers} = "
              f"{r * spec.layers:.3f} ms; outside routers {ms - r * spec.layers:.3f} ms", flush=True)
    del pipe
    gc.collect()
    torch.cuda.empty_cache()
