"""Device timeline of the single-layer (decode) step's main-stream chain at the
Qwen3 shape: CUDA events between router, layout and scoring, with a device sleep
queued first so the launches are timed on the GPU, not at the host's rate."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

spec = spec_for(sys.argv[1] if len(sys.argv) > 1 else "qwen3")
eng = mp.Engine(0)
pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
s, D = spec, spec.groups
N = 50


def chain():
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    evs[0].record()
    eng.router_topk(pipe.X[0], pipe.model.W[0], s.top_k, s.score_fn, s.renorm, out=(pipe.idx, pipe.w))
    evs[1].record()
    eng.dispatch_layout(pipe.idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok, n_tags=s.domains,
                        demand=pipe.dem_cl[0], tag_pop=pipe.pop, perm_out=(pipe.sp, pipe.pp, pipe.ko),
                        src2=pipe.src_rr, demand2=pipe.dem_rr[0])
    evs[2].record()
    eng.coactivation(pipe.idx, s.experts, out=pipe.coact)
    evs[3].record()
    eng.score_and_finalize(pipe.dem_cl, pipe.luts_cl, pipe.g2n, D, pipe.cost, pipe.topology,
                           row_node=pipe.g2n, out=pipe.sc_cl, fin_out=pipe.fin_cl[0],
                           payload=pipe.fin_cl[1])
    evs[4].record()
    return evs


for _ in range(5):
    chain()
torch.cuda.synchronize()
torch.cuda._sleep(int(5e8))
runs = [chain() for _ in range(N)]
torch.cuda.synchronize()
names = ["router", "layout (K2+K3)", "coactivation (K4)", "score (K5)"]
tot = [0.0] * 4
for e in runs:
    for i in range(4):
        tot[i] += e[i].elapsed_time(e[i + 1]) * 1e3
print(f"{spec.name}: " + ", ".join(f"{n} {t / N:.1f} us" for n, t in zip(names, tot)) +
      f"; chain {sum(tot) / N:.1f} us")
pipe.plan.capture()
for _ in range(3):
    pipe.plan.run(3)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(5e8))
a.record()
for _ in range(N):
    pipe.plan.run(3)
b.record()
torch.cuda.synchronize()
print(f"graphed step {a.elapsed_time(b) / N * 1e3:.1f} us")
