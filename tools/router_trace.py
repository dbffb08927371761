"""Phase breakdown of one router launch from an experiment build with
-DMPB_ROUTER_TRACE (tools/build_exp.sh rtrace -DMPB_ROUTER_TRACE=1;
MPB_LIB_PATH=exp_libs/rtrace.so python tools/router_trace.py --T 4096 ...):
per-CTA %globaltimer stamps, reported relative to the earliest entry."""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23150_b200 import _abi, moeplace as mp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=4096)
ap.add_argument("--H", type=int, default=4096)
ap.add_argument("--E", type=int, default=128)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--fn", type=int, default=0)
ap.add_argument("--layers", type=int, default=0)
a, _ = ap.parse_known_args()
eng = mp.Engine(0)
X = torch.randn(a.T, a.H, device="cuda").to(torch.bfloat16)
W = (torch.randn(a.E, a.H, device="cuda") / a.H ** 0.5).to(torch.bfloat16)
for _ in range(3):
    if a.layers:
        eng.router_topk_layers([X] * a.layers, [W] * a.layers, a.k, a.fn, True)
    else:
        eng.router_topk(X, W, a.k, a.fn, True)
torch.cuda.synchronize()
assert _abi.lib().mpb_debug_router_trace(None, 0) == 0
if a.layers:  # one traced launch on an idle GPU
    eng.router_topk_layers([X] * a.layers, [W] * a.layers, a.k, a.fn, True)
else:
    eng.router_topk(X, W, a.k, a.fn, True)
torch.cuda.synchronize()
n = 2 * 148 * 16
buf = (C.c_ulonglong * n)()
assert _abi.lib().mpb_debug_router_trace(buf, n) == 0
t = np.array(buf, dtype=np.uint64).reshape(-1, 16)
used = t[:, 0] > 0
t = t[used].astype(np.int64)
t0 = t[:, 0].min()
names = ["entry", "pdl_wait", "first_tma", "last_commit", "acc_ready", "summed", "epi_done",
         "exit", None, None, "pass1", "pass2", "merged", "softmax", "peers_free", "rx_landed"]
roles = t[:, 8]
if "--by-part" in sys.argv:  # cluster tail: group by K part (cluster rank) instead of role
    roles = np.nonzero(used)[0] % 4

print(f"T={a.T} H={a.H} E={a.E} k={a.k} layers={a.layers}: {used.sum()} CTAs; "
      f"items/CTA {np.bincount(t[:, 9]).nonzero()[0].tolist()}")
for r in sorted(set(roles.tolist())):
    sel = t[roles == r]
    line = " ".join(f"{nm}={np.median(sel[sel[:, i] > 0, i] - t0) / 1e3:6.2f}us"
                    for i, nm in enumerate(names) if nm and (sel[:, i] > 0).sum() * 2 > len(sel))
    print(f"role {r} ({len(sel)} CTAs, medians): {line}")
print(f"kernel span {(t[:, 7].max() - t0) / 1e3:.2f} us")
ep = t[t[:, 10] > 0]
print(f"scan (warp 4 lane 0, medians over CTAs): tmem-load cycles {np.median(ep[:, 13]):.0f}, "
      f"insertion cycles {np.median(ep[:, 14]):.0f}, hits {np.median(ep[:, 15]):.0f}")
for r in sorted(set(roles.tolist())):
    row = t[roles == r][0]
    print(f"  e.g. role {r}:", [round((v - t0) / 1e3, 2) if v > 0 else None for v in row[:16]])
