"""Where the DSv3 step's non-router time goes: the graphed step timed with
parts of the side stream's statistics work switched off (experiment only —
the switched-off variants do not produce the step's full results).
  python tools/step_probe.py [variant ...]   variants: full, nocoact, noscore"""
import gc
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

eng = mp.Engine(0)
for v in sys.argv[1:] or ["full", "nocoact", "noscore"]:
    over = {"coact": False} if v == "nocoact" else {}
    os.environ["MPB_SCORE_PER_CHUNK"] = "0" if v == "noscore" else "1"
    spec = spec_for("dsv3", **over)
    pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
    for _ in range(2):
        pipe.step()
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
