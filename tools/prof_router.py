"""Runs the router GEMM + top-k alone for profiling (ncu / timing)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=65536)
ap.add_argument("--H", type=int, default=7168)
ap.add_argument("--E", type=int, default=256)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--fn", type=int, default=1)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--sms", type=int, default=0, help="SM budget (0 = all)")
ap.add_argument("--nx", type=int, default=1, help="distinct X / W buffers rotated per launch")
ap.add_argument("--events", action="store_true", help="an event pair around every launch")
ap.add_argument("--layers", type=int, default=0,
                help="time one grouped launch over this many layers (mpb_router_topk_layers); "
                     "reported per layer")
ap.add_argument("--sleep", type=float, default=0.0,
                help="ms of device sleep queued before the timed launches, so small-T launches are "
                     "timed on the GPU rather than at the host's launch rate")
a = ap.parse_args()
eng = mp.Engine(0)
if a.sms:
    eng.set_sm_budget(a.sms)
Xs = [torch.randn(a.T, a.H, device="cuda").to(torch.bfloat16) for _ in range(a.nx)]
Ws = [(torch.randn(a.E, a.H, device="cuda") / a.H ** 0.5).to(torch.bfloat16) for _ in range(a.nx)]
X, W = Xs[0], Ws[0]
if a.layers:
    LX = [X] * a.layers if a.nx == 1 else [Xs[i % a.nx] for i in range(a.layers)]
    LW = [W] * a.layers if a.nx == 1 else [Ws[i % a.nx] for i in range(a.layers)]
    lout = (torch.empty(a.layers, a.T, a.k, dtype=torch.int32, device="cuda"),
            torch.empty(a.layers, a.T, a.k, dtype=torch.float32, device="cuda"))
    for _ in range(2):
        eng.router_topk_layers(LX, LW, a.k, a.fn, True, out=lout)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(a.iters):
        eng.router_topk_layers(LX, LW, a.k, a.fn, True, out=lout)
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / a.iters / a.layers
    print(f"grouped router x{a.layers} T={a.T} H={a.H} E={a.E} k={a.k}: {ms:.4f} ms/layer  "
          f"{2 * a.T * a.H * a.E / ms / 1e9:.1f} TFLOP/s  {(a.T * a.H * 2) / ms / 1e6:.0f} GB/s(X)")
out = (torch.empty(a.T, a.k, dtype=torch.int32, device="cuda"),
       torch.empty(a.T, a.k, dtype=torch.float32, device="cuda"))
for _ in range(2):
    eng.router_topk(X, W, a.k, a.fn, True, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cycles = int(a.sleep * 1e-3 * torch.cuda.get_device_properties(0).clock_rate * 1e3)
if cycles:
    torch.cuda._sleep(cycles)
s.record()
pairs = []
for i in range(a.iters):
    if a.events:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    eng.router_topk(Xs[i % a.nx], Ws[i % a.nx], a.k, a.fn, True, out=out)
    if a.events:
        e1.record()
        pairs.append((e0, e1))
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.iters
if pairs:
    print(f"per-launch events: {sum(x.elapsed_time(y) for x, y in pairs) / len(pairs):.4f} ms")
tf = 2 * a.T * a.H * a.E / ms / 1e9
print(f"router T={a.T} H={a.H} E={a.E} k={a.k}: {ms:.4f} ms  {tf:.1f} TFLOP/s  "
      f"{(a.T * a.H * 2) / ms / 1e6:.0f} GB/s(X)")
# cuBLAS reference point for the same GEMM (library baseline, not on the path)
C = torch.empty(a.T, a.E, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    torch.matmul(X, W.t(), out=C)
torch.cuda.synchronize()
if cycles:
    torch.cuda._sleep(cycles)
s.record()
for _ in range(a.iters):
    torch.matmul(X, W.t(), out=C)
e.record()
torch.cuda.synchronize()
ms2 = s.elapsed_time(e) / a.iters
print(f"cublas bf16 GEMM same shape: {ms2:.4f} ms  {2 * a.T * a.H * a.E / ms2 / 1e9:.1f} TFLOP/s")
