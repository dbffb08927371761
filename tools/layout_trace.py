"""Phase stamps of the single-cluster layout kernel (experiment build with
-DMPB_LAYOUT_TRACE, loaded through MPB_LIB_PATH):

    tools/build_exp.sh lctrace -DMPB_LAYOUT_TRACE=1
    MPB_LIB_PATH=exp_libs/lctrace.so python tools/layout_trace.py [workload]

Prints, per phase, the min / median / max over the cluster's CTAs of the
%globaltimer stamp relative to the earliest kernel entry (ns), for one
isolated launch and for the last of 20 back-to-back launches."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23150_b200 import _abi  # noqa: E402
from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402

PH = ["entry", "cluster bar", "pdl wait", "warp0 ph1", "all ph1", "flush", "bar 2", "exit"]
w = sys.argv[1] if len(sys.argv) > 1 else "qwen3"
eng = mp.Engine(0)
pipe = RoutingPipeline(spec_for(w), eng, 0, 1, resident=True)
pipe.step()
torch.cuda.synchronize()
s = pipe.spec
lib = _abi.lib()
fn = lib.mpb_debug_layout_trace
fn.argtypes = [C.c_void_p]


def call():
    eng.dispatch_layout(pipe.idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok,
                        n_tags=s.domains, demand=pipe.dem_cl[0], tag_pop=pipe.pop,
                        perm_out=(pipe.sp, pipe.pp, pipe.ko), src2=pipe.src_rr,
                        demand2=pipe.dem_rr[0])


def show(title):
    buf = np.zeros(16 * 8, np.uint64)
    assert fn(buf.ctypes.data) == 0
    t = buf.reshape(16, 8).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    print(f"{title}: {len(t)} CTAs")
    for i, name in enumerate(PH):
        col = t[:, i] - t0
        print(f"  {name:12s} min {col.min():7d}  med {int(np.median(col)):7d}  max {col.max():7d} ns")


for _ in range(3):
    call()
    torch.cuda.synchronize()
show("isolated launch")
with torch.cuda.stream(eng.stream):
    torch.cuda._sleep(int(5e7))
for _ in range(20):
    call()
torch.cuda.synchronize()
show("last of 20 back-to-back")
