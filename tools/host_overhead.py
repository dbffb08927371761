"""Host-side enqueue cost of the step's ABI calls (the GPU is kept busy by a
long sleep kernel, so every call returns as soon as it has enqueued its work):
microseconds of host time per call, at the Qwen3 decode shape."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

spec = spec_for("qwen3")
eng = mp.Engine(0)
pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
pipe.step()
torch.cuda.synchronize()
s, D = spec, spec.groups
N = 50
cases = {
    "plan.run(LAYERS|SCORE)": lambda: pipe.plan.run(3),
    "plan.run(LAYERS)": lambda: pipe.plan.run(1),
    "router_topk": lambda: eng.router_topk(pipe.X[0], pipe.model.W[0], s.top_k, s.score_fn,
                                           s.renorm, out=(pipe.idx, pipe.w)),
    "dispatch_layout": lambda: eng.dispatch_layout(
        pipe.idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok, n_tags=s.domains,
        demand=pipe.dem_cl[0], tag_pop=pipe.pop, perm_out=(pipe.sp, pipe.pp, pipe.ko),
        src2=pipe.src_rr, demand2=pipe.dem_rr[0]),
    "coactivation": lambda: eng.coactivation(pipe.idx, s.experts, out=pipe.coact),
    "score_and_finalize": lambda: eng.score_and_finalize(
        pipe.dem_cl, pipe.luts_cl, pipe.g2n, D, pipe.cost, pipe.topology, row_node=pipe.g2n,
        out=pipe.sc_cl, fin_out=pipe.fin_cl[0], payload=pipe.fin_cl[1]),
}
for name, fn in cases.items():
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e9))  # ~1 s of GPU work ahead of the calls
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    dt = (time.perf_counter() - t0) / N
    torch.cuda.synchronize()
    print(f"{name:26s} {dt * 1e6:8.1f} us host per call")
