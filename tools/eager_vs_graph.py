"""Eager vs graph-replayed C++ step at the Qwen3 shape: device time per step
(CUDA events over N back-to-back runs), with and without a device sleep
queued ahead (pre-queued: the GPU's own execution time; not pre-queued: the
host's enqueue rate included)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "qwen3"
spec = spec_for(wl)
eng = mp.Engine(0)
pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
N = 50 if wl == "qwen3" else 5


def timed(prequeue):
    for _ in range(3):
        pipe.plan.run(3)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if prequeue:
        torch.cuda._sleep(int(5e8))
    s.record()
    for _ in range(N):
        pipe.plan.run(3)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / N * 1e3


print(f"{wl} eager   : {timed(False):8.1f} us/step (host-paced)  {timed(True):8.1f} us/step (pre-queued)")
pipe.plan.capture()
print(f"{wl} graphed : {timed(False):8.1f} us/step (host-paced)  {timed(True):8.1f} us/step (pre-queued)")
