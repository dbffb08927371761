"""K2/K3 (dispatch_layout: histograms + stable permutation) warm timings at the
BASELINE shapes, on the pipeline's own routed idx and metadata (the exact call
of RoutingPipeline._layer_tail), CUDA events over launches pre-queued behind a sleep kernel.

    python tools/layout_bench.py [qwen3 dsv3 domain maverick] [--once]

--once: each case launched once after a warm-up (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

ONCE = "--once" in sys.argv
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["qwen3", "dsv3", "domain"]
eng = mp.Engine(0)
for w in names:
    spec = spec_for(w, layers=1) if w == "dsv3" else spec_for(w)
    pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
    pipe.step()
    torch.cuda.synchronize()
    s = spec

    def full():
        eng.dispatch_layout(pipe.idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok,
                            n_tags=s.domains, demand=pipe.dem_cl[0], tag_pop=pipe.pop,
                            perm_out=(pipe.sp, pipe.pp, pipe.ko), src2=pipe.src_rr,
                            demand2=pipe.dem_rr[0])

    def counts():
        eng.dispatch_layout(pipe.idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok,
                            n_tags=s.domains, demand=pipe.dem_cl[0], tag_pop=pipe.pop,
                            permutation=False, src2=pipe.src_rr, demand2=pipe.dem_rr[0])

    T, k = pipe.idx.shape
    for name, fn in (("layout+perm", full), ("layout counts", counts)):
        fn()
        torch.cuda.synchronize()
        if ONCE:
            continue
        n = 50 if T * k <= 1 << 20 else 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = eng.launches
        # keep the GPU busy while the host queues the calls: the events time the
        # kernels, not the host's enqueue rate
        with torch.cuda.stream(eng.stream):
            torch.cuda._sleep(int(5e7))
        e0.record(eng.stream)
        for _ in range(n):
            fn()
        e1.record(eng.stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        launches = (eng.launches - l0) // n
        byts = T * k * (4 + (8 if name == "layout+perm" else 0)) + T * 4
        print(f"{w:9s} T={T:8d} k={k} E={s.experts:3d} {name:14s} {us:8.2f} us "
              f"({launches} launches)  {byts / us / 1e3:8.1f} GB/s algorithmic")
    del pipe
    torch.cuda.empty_cache()
