import sys, traceback
sys.path.insert(0, "/root/repo")
import torch
from paper_2604_23150_b200 import moeplace as mp
from paper_2604_23150_b200.pipeline import RoutingPipeline, WorkloadSpec, spec_for
for spec in [WorkloadSpec("tiny1", 1, 4096, 512, 128, 8, 0, True, groups=8, nodes=2, domains=8, preferred=16, candidates=64), spec_for("dsv3", layers=12, tokens=16384)]:
    eng = mp.Engine(0)
    pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
    for _ in range(3):
        pipe.step()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(eng.stream); pipe.step(); e.record(eng.stream); torch.cuda.synchronize()
    r = pipe.router_ms()
    print(spec.name, "step ms", s.elapsed_time(e), "sum router ms", sum(r), "chunks", pipe.plan.chunks())
    try:
        pipe.plan.capture()
        print("capture ok")
    except Exception as ex:
        traceback.print_exc()
