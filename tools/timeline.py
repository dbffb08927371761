"""Per-layer device timeline of one DSv3 step (CUDA events on both streams):
router, layout (main stream), co-activation (side stream), join, gaps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import WORKLOADS, RoutingPipeline  # noqa: E402

spec = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "dsv3"]
eng = mp.Engine(0)
pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
for _ in range(3):
    pipe.step()
torch.cuda.synchronize()
s, side = spec, pipe.side
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
rows = []
pipe.stats.zero_()
t0 = ev()
t0.record(eng.stream)
for l in range(s.layers):
    r0, r1, l1, c1, j1 = ev(), ev(), ev(), ev(), ev()
    r0.record(eng.stream)
    eng.router_topk(pipe.X[l], pipe.model.W[l], s.top_k, s.score_fn, s.renorm,
                    out=(pipe.idx, pipe.w))
    r1.record(eng.stream)
    if side is not None:
        side.stream.wait_event(r1)
        side.coactivation(pipe.idx, s.experts, out=pipe.coact)
        c1.record(side.stream)
    eng.dispatch_layout(pipe.idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok,
                        n_tags=s.domains, demand=pipe.dem_cl[l], tag_pop=pipe.pop,
                        perm_out=(pipe.sp, pipe.pp, pipe.ko), src2=pipe.src_rr,
                        demand2=pipe.dem_rr[l])
    l1.record(eng.stream)
    if side is not None:
        eng.stream.wait_event(c1)
    j1.record(eng.stream)
    rows.append((r0, r1, l1, c1 if side is not None else None, j1))
e0 = ev()
e0.record(eng.stream)
pipe._score_only()
e1 = ev()
e1.record(eng.stream)
torch.cuda.synchronize()
router = [a.elapsed_time(b) * 1e3 for a, b, *_ in rows]
layout = [b.elapsed_time(c) * 1e3 for a, b, c, *_ in rows]
coact = [b.elapsed_time(d) * 1e3 for a, b, c, d, e in rows if d is not None]
tail = [b.elapsed_time(e) * 1e3 for a, b, c, d, e in rows]
gap = [rows[i][4].elapsed_time(rows[i + 1][0]) * 1e3 for i in range(len(rows) - 1)]
total = t0.elapsed_time(e1) * 1e3
med = lambda v: float(np.median(v)) if v else float("nan")  # noqa: E731
print(f"step {total:.0f} us  ({s.layers} layers; scoring {e0.elapsed_time(e1) * 1e3:.0f} us)")
print(f"per layer (median us): router {med(router):.1f}  layout {med(layout):.1f}  "
      f"coact(side) {med(coact):.1f}  router-end->join {med(tail):.1f}  join->next router "
      f"{med(gap):.1f}")
print(f"sum over layers (us): router {sum(router):.0f}  tail {sum(tail):.0f}  gaps {sum(gap):.0f}")
