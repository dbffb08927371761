"""Interleaved A/B of step-schedule knobs on ONE pipeline (DSv3 shape): the
plan is rebuilt per variant and the variants alternate round by round, so the
box's power-cap drift hits them alike. Experiments only.
  python tools/step_ab.py [rounds]"""
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

VARIANTS = {  # name: (env, pipeline attributes); measured this round, all within about 2%
    "base": ({}, {}),
    "side16": ({}, {"side_sms": 16}),
    "group12": ({}, {"router_group": 12}),
    "lbatch8": ({"MPB_LAYOUT_BATCH": "8"}, {}),
    "tailboost2": ({"MPB_TAIL_BOOST": "2"}, {}),
}
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = mp.Engine(0)
pipe = RoutingPipeline(spec_for("dsv3"), eng, 0, 1, resident=True)
base_attrs = {"router_group": pipe.router_group, "side_sms": pipe.side_sms}
res = {k: [] for k in VARIANTS}
for r in range(rounds):
    for name, (env, attrs) in VARIANTS.items():
        for k in ("MPB_TAIL_BOOST", "MPB_MAIN_TAIL_CHUNKS", "MPB_LAYOUT_BATCH"):
            os.environ.pop(k, None)
        os.environ.update(env)
        for k, v in {**base_attrs, **attrs}.items():
            setattr(pipe, k, v)
        pipe.plan = None
        torch.cuda.synchronize()
        pipe._build_plan()
        pipe.step()
        assert pipe.capture()
        for _ in range(2):
            pipe.step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        for _ in range(6):
            pipe.step()
        b.record(eng.stream)
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / 6)
        print(f"round {r} {name:10s} {res[name][-1]:.3f} ms", flush=True)
base = statistics.mean(res["base"])
for name, v in res.items():
    m = statistics.mean(v)
    print(f"{name:10s} mean {m:.3f} ms  ({(m / base - 1) * 100:+.1f}% vs base)  runs {[round(x, 3) for x in v]}")
