"""GPU parity of the tcgen05 router GEMM + fused top-k (K1).

Logits (bf16 inputs, fp32 accumulate on tensor cores) vs a float64 CPU-free
torch reference of the same bf16 inputs: |err| <= 1e-4 * sqrt(H) * rms(x) *
rms(w) + 1e-5 (accumulation-order tolerance of an fp32 dot product of length
H). Indices must equal the oracle's top-k on the SAME device logits
(bit-exact, lowest-id tie rule); weights within 2e-6 relative."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return mp.Engine(0)


CASES = [  # T, H, E, k, score_fn, renorm
    (128, 64, 64, 2, 0, False), (1000, 512, 128, 8, 0, True), (4096, 4096, 128, 8, 0, False),
    (2048, 7168, 256, 8, 1, True), (3001, 5120, 128, 1, 1, False), (257, 1024, 256, 16, 0, True),
    (65536, 7168, 256, 8, 1, True),
    # E not a tile width: padded to 64 / 128 / 256 with masked columns
    (4096, 1024, 160, 8, 1, True), (3000, 512, 96, 6, 0, False), (2048, 768, 32, 2, 0, True),
    (1000, 256, 8, 2, 0, False), (5000, 2048, 200, 16, 1, True), (777, 128, 1, 1, 1, False)]


@pytest.mark.parametrize("case", CASES)
def test_router_topk(eng, oracle, case):
    T, H, E, k, fn, renorm = case
    g = torch.Generator(device="cuda").manual_seed(T + H + E)
    X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    idx, w, logits = eng.router_topk(X, W, k, fn, renorm, want_logits=True)
    torch.cuda.synchronize()
    ref = X.double() @ W.double().t()
    tol = 1e-4 * H ** 0.5 * float(X.float().pow(2).mean().sqrt()) * \
        float(W.float().pow(2).mean().sqrt()) + 1e-5
    err = (logits.double() - ref).abs().max().item()
    assert err <= tol, (err, tol)
    lg = logits.cpu().numpy()
    sel = slice(None) if T <= 8192 else slice(0, 8192)
    ri, rw = oracle.topk_logits(lg[sel], k, fn, renorm)
    np.testing.assert_array_equal(idx.cpu().numpy()[sel], ri)
    np.testing.assert_allclose(w.cpu().numpy()[sel], rw, rtol=2e-6, atol=1e-7)
    # without materialising logits the routing is identical
    idx2, w2 = eng.router_topk(X, W, k, fn, renorm)
    assert torch.equal(idx2, idx) and torch.equal(w2, w)


def test_router_ties_lowest_id(eng):
    # identical expert rows -> identical logits -> lowest ids win
    T, H, E, k = 256, 128, 64, 4
    X = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    W = torch.randn(1, H, device="cuda").to(torch.bfloat16).repeat(E, 1)
    idx, _ = eng.router_topk(X, W, k, 0, False)
    torch.cuda.synchronize()
    assert (idx.cpu() == torch.arange(k, dtype=torch.int32)).all()


def test_router_and_coact_graph_replay(eng):
    """Captured once, replayed on new inputs: the router's split-K tail flags and
    the co-activation grid barrier are self-resetting, so every replay matches
    an eager run (DSv3 shape: exercises the split tail)."""
    T, H, E, k = 65536, 7168, 256, 8
    g = torch.Generator(device="cuda").manual_seed(5)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    X = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    w = torch.empty(T, k, dtype=torch.float32, device="cuda")
    co = torch.zeros(E, E, dtype=torch.uint64, device="cuda")
    s = torch.cuda.Stream()
    geng = mp.Engine(0, stream=s)
    X.copy_(torch.randn(T, H, device="cuda", generator=g))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):  # warm-up (allocates scratch) outside capture
        geng.router_topk(X, W, k, 1, True, out=(idx, w))
        geng.coactivation(idx, E, out=co)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        co.zero_()
        geng.router_topk(X, W, k, 1, True, out=(idx, w))
        geng.coactivation(idx, E, out=co)
    for rep in range(3):
        X.copy_(torch.randn(T, H, device="cuda", generator=g))
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        ri, rw = eng.router_topk(X, W, k, 1, True)
        rc = eng.coactivation(ri, E)
        torch.cuda.synchronize()
        assert torch.equal(idx, ri) and torch.equal(w, rw), rep
        assert torch.equal(co, rc), rep


def test_sm_budget_changes_nothing_but_the_grid(eng):
    """Contexts sized for fewer SMs (the overlapped schedule: router on 128,
    statistics on 20): the router's logits stay within the fp32
    accumulation-order bound (the split-K tail of the last wave depends on the
    unit count), its top-k equals the oracle's on the budgeted logits, and the
    integer kernels (co-activation) are bit-identical."""
    T, H, E, k = 65536, 1024, 256, 8
    g = torch.Generator(device="cuda").manual_seed(9)
    X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    full = mp.Engine(0)
    ref_idx, ref_w, ref_logits = full.router_topk(X, W, k, 1, True, want_logits=True)
    ref_c = full.coactivation(ref_idx, E)
    tol = 1e-4 * H ** 0.5 * float(X.float().pow(2).mean().sqrt()) * \
        float(W.float().pow(2).mean().sqrt()) + 1e-5
    for sms in (128, 20, 2):
        e = mp.Engine(0)
        e.set_sm_budget(sms)
        idx, w, logits = e.router_topk(X, W, k, 1, True, want_logits=True)
        c = e.coactivation(ref_idx, E)
        torch.cuda.synchronize()
        assert (logits - ref_logits).abs().max().item() <= tol, sms
        ti, tw = e.topk_logits(logits, k, 1, True)
        assert torch.equal(ti, idx) and torch.equal(tw, w), sms
        assert torch.equal(c, ref_c), sms


@pytest.mark.parametrize("shape", [(4096, 4096, 128, 8, 0, False), (1024, 7168, 256, 8, 1, True),
                                   (300, 1088, 64, 4, 0, True)])
def test_router_split_k_parts(eng, oracle, shape, monkeypatch):
    """Small decode batches (fewer tiles than SMs) split every tile's K range
    over up to 4 units (router.cu next_item / launch_router_n). Whatever the
    number of parts (uneven ones included: 1088 / 64 = 17 k-steps), the logits
    stay within the fp32 accumulation-order bound of the float64 reference and
    the top-k is the oracle's on the same logits; the partial flags reset
    themselves, so back-to-back launches with different splits stay correct."""
    T, H, E, k, fn, renorm = shape
    g = torch.Generator(device="cuda").manual_seed(T * 7 + H)
    X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    ref = X.double() @ W.double().t()
    tol = 1e-4 * H ** 0.5 * float(X.float().pow(2).mean().sqrt()) * \
        float(W.float().pow(2).mean().sqrt()) + 1e-5
    for cap in ("1", "2", "3", "8", "8", "2"):
        monkeypatch.setenv("MPB_ROUTER_MAX_SPLITS", cap)
        idx, w, logits = eng.router_topk(X, W, k, fn, renorm, want_logits=True)
        torch.cuda.synchronize()
        assert (logits.double() - ref).abs().max().item() <= tol, cap
        ri, rw = oracle.topk_logits(logits.cpu().numpy(), k, fn, renorm)
        np.testing.assert_array_equal(idx.cpu().numpy(), ri)
        np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("shape", [(4096, 4096, 128, 8, 0, True), (4096, 4096, 128, 1, 1, False),
                                   (2048, 1024, 64, 4, 0, False), (1000, 2048, 96, 6, 1, True),
                                   (3000, 512, 128, 16, 0, True), (4096, 2048, 256, 8, 1, True),
                                   # 60 tiles -> 2 K parts (64-row shares, 4 threads per row)
                                   (7680, 2048, 128, 8, 0, True), (7000, 1024, 64, 16, 1, False),
                                   (1024, 512, 64, 16, 0, True)])
def test_router_cluster_tail_equals_global_tail(eng, oracle, shape, monkeypatch):
    """Single-CTA tiles run the split-K tail through distributed shared memory
    (the K parts of a tile in one cluster, reduce-scatter of the partials with
    st.async, top-k of each CTA's row share by all 8 epilogue warps). The
    partials are summed in the same K-part order as the global-memory tail
    (MPB_ROUTER_GLOBAL_TAIL=1), so the logits are bit-identical, the indices
    are the oracle's top-k of those logits and the weights agree with it; the
    256-expert case runs single-CTA tiles (MPB_ROUTER_SINGLE=1)."""
    T, H, E, k, fn, renorm = shape
    if E > 128:
        monkeypatch.setenv("MPB_ROUTER_SINGLE", "1")
    g = torch.Generator(device="cuda").manual_seed(T * 3 + E)
    X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    out = {}
    for tail in ("global", "cluster", "cluster"):
        if tail == "global":
            monkeypatch.setenv("MPB_ROUTER_GLOBAL_TAIL", "1")
        else:
            monkeypatch.delenv("MPB_ROUTER_GLOBAL_TAIL", raising=False)
        out[tail] = eng.router_topk(X, W, k, fn, renorm, want_logits=True)
        torch.cuda.synchronize()
    (gi, gw, gl), (ci, cw, cl) = out["global"], out["cluster"]
    assert torch.equal(gl, cl)
    ri, rw = oracle.topk_logits(cl.cpu().numpy(), k, fn, renorm)
    np.testing.assert_array_equal(ci.cpu().numpy(), ri)
    np.testing.assert_array_equal(gi.cpu().numpy(), ri)
    np.testing.assert_allclose(cw.cpu().numpy(), rw, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("shape", [(3, 5000, 1024, 256, 8, 1, True), (4, 4096, 4096, 128, 8, 0, False),
                                   (2, 300, 512, 64, 4, 0, True), (5, 65536, 7168, 256, 8, 1, True)])
def test_router_topk_layers_matches_per_layer(eng, shape, monkeypatch):
    """One grouped launch over L layers (mpb_router_topk_layers) == L single
    launches. Without the split-K tail every tile accumulates its K range in
    the same order in both, so idx / w are bit-identical; with it, only the
    last wave's tiles differ in fp32 summation order (near-tie flips only)."""
    L, T, H, E, k, fn, renorm = shape
    g = torch.Generator(device="cuda").manual_seed(L * T + H)
    Xs = [torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    Ws = [(torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
          for _ in range(L)]
    monkeypatch.setenv("MPB_ROUTER_NO_SPLIT", "1")
    ref = [eng.router_topk(X, W, k, fn, renorm) for X, W in zip(Xs, Ws)]
    idx, w = eng.router_topk_layers(Xs, Ws, k, fn, renorm)
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(idx[l], ref[l][0]), l
        assert torch.equal(w[l], ref[l][1]), l
    monkeypatch.delenv("MPB_ROUTER_NO_SPLIT")
    idx2, w2 = eng.router_topk_layers(Xs, Ws, k, fn, renorm)
    ref2 = [eng.router_topk(X, W, k, fn, renorm) for X, W in zip(Xs, Ws)]
    torch.cuda.synchronize()
    for l in range(L):
        same = (idx2[l] == ref2[l][0]).all(1)
        assert same.float().mean().item() >= 0.999, l
        # weights follow logits that differ by fp32 summation order (|dlogit| ~
        # 1e-5 at H = 4096): relative weight error of the same order
        torch.testing.assert_close(w2[l][same], ref2[l][1][same], rtol=2e-4, atol=1e-6)
    # the descriptor table is cached: a second call with the same buffers reuses it
    idx3, w3 = eng.router_topk_layers(Xs, Ws, k, fn, renorm)
    assert torch.equal(idx3, idx2) and torch.equal(w3, w2)


def test_router_topk_layers_errors(eng):
    """Grouped-launch argument checks map onto the reference's error classes:
    NULL buffers -> ValidationError, misaligned / unsupported shapes ->
    ConfigError; zero layers is a no-op; a second descriptor table for new
    buffers is created next to the first (both stay valid)."""
    import ctypes as C

    from paper_2604_23150_b200 import _abi
    from paper_2604_23150_b200.errors import ConfigError, ValidationError
    T, H, E, k = 512, 256, 64, 4
    Xs = [torch.randn(T, H, device="cuda").to(torch.bfloat16) for _ in range(2)]
    Ws = [(torch.randn(E, H, device="cuda") / 16).to(torch.bfloat16) for _ in range(2)]
    idx = torch.empty(2, T, k, dtype=torch.int32, device="cuda")
    w = torch.empty(2, T, k, dtype=torch.float32, device="cuda")
    xp = (C.c_void_p * 2)(Xs[0].data_ptr(), 0)
    wp = (C.c_void_p * 2)(Ws[0].data_ptr(), Ws[1].data_ptr())
    with pytest.raises(ValidationError):
        _abi.call("mpb_router_topk_layers", eng.ctx, 2, xp, wp, T, H, E, k, 0, 0,
                  C.c_void_p(idx.data_ptr()), C.c_void_p(w.data_ptr()), None)
    xp = (C.c_void_p * 2)(Xs[0].data_ptr() + 2, Xs[1].data_ptr())
    with pytest.raises(ConfigError):
        _abi.call("mpb_router_topk_layers", eng.ctx, 2, xp, wp, T, H, E, k, 0, 0,
                  C.c_void_p(idx.data_ptr()), C.c_void_p(w.data_ptr()), None)
    with pytest.raises(ConfigError):  # H not a multiple of 64
        _abi.call("mpb_router_topk_layers", eng.ctx, 2, xp, wp, T, H - 32, E, k, 0, 0,
                  C.c_void_p(idx.data_ptr()), C.c_void_p(w.data_ptr()), None)
    _abi.call("mpb_router_topk_layers", eng.ctx, 0, None, None, T, H, E, k, 0, 0, None, None, None)
    a = eng.router_topk_layers(Xs, Ws, k, 0, False)
    b = eng.router_topk_layers(Xs[::-1], Ws[::-1], k, 0, False)
    c = eng.router_topk_layers(Xs, Ws, k, 0, False)
    torch.cuda.synchronize()
    assert torch.equal(a[0], c[0]) and torch.equal(a[0][0], b[0][1]) and torch.equal(a[0][1], b[0][0])


@pytest.mark.parametrize("sms", [148, 64, 20, 8])
def test_cluster_tail_under_sm_budgets(oracle, sms):
    """The decode-shape router (single-CTA tiles, split-K tail through
    distributed shared memory) in contexts sized for fewer SMs: the unit count,
    the K split and the resident-cluster cap all change, the top-k stays the
    oracle's on the launch's own logits and the weights agree with it."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, H, E, k = 4096, 4096, 128, 8
    g = torch.Generator(device="cuda").manual_seed(sms)
    X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    e = mp.Engine(0)
    e.set_sm_budget(sms)
    for fn in (0, 1):
        idx, w, logits = e.router_topk(X, W, k, fn, True, want_logits=True)
        torch.cuda.synchronize()
        ri, rw = oracle.topk_logits(logits.cpu().numpy(), k, fn, True)
        np.testing.assert_array_equal(idx.cpu().numpy(), ri)
        np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("tail", ["cluster", "global", "none"])
@pytest.mark.parametrize("shape", [(4096, 1024, 128, 8, 0), (4096, 1024, 128, 16, 1), (2048, 512, 64, 16, 0),
                                   # E = 256: 2-SM CTA pairs (UMMA M=256), global split tail
                                   (8192, 1024, 256, 8, 1)])
def test_router_ties_inf_nan(eng, oracle, shape, tail, monkeypatch):
    """Non-finite and tied logits follow the oracle's order on every epilogue
    (cluster tail, global split tail, no split): real values (+-inf included)
    descend, equal logits keep the lower expert id (duplicated W rows give
    bit-equal columns), -0 ties +0, -inf fills before NaN, NaN last in id
    order. Rows with X[t, 0] = +-inf make +-inf / NaN logits through W[:, 0]."""
    T, H, E, k, fn = shape
    g = torch.Generator(device="cuda").manual_seed(T + E + k)
    X = torch.randn(T, H, device="cuda", generator=g)
    W = torch.randn(E, H, device="cuda", generator=g) / H ** 0.5
    W[:, 0] = W[:, 0].abs() + 0.01
    W[2, 0] = W[E - 14, 0] = -0.5       # X = -inf rows: +inf here, -inf elsewhere
    W[5, 0] = W[9, 0] = W[E - 51, 0] = 0.0  # inf * 0 -> NaN
    W[E // 2:E // 2 + 8, 0] = 0.0         # a NaN-heavy block
    W[7] = W[3]                           # exact ties on normal rows
    W[E - 1] = W[3]
    W[E - 20, 1:] = W[11, 1:]
    X[1::7, 0] = float("inf")
    X[3::7, 0] = -float("inf")
    X[5::7, 0] = 0.0
    X[5::7, 1:] = 0.0                     # an all-zero row: every logit +-0, all ties
    X, W = X.to(torch.bfloat16), W.to(torch.bfloat16)
    if tail == "global":
        monkeypatch.setenv("MPB_ROUTER_GLOBAL_TAIL", "1")
    elif tail == "none":
        monkeypatch.setenv("MPB_ROUTER_NO_SPLIT", "1")
    idx, w, logits = eng.router_topk(X, W, k, fn, True, want_logits=True)
    torch.cuda.synchronize()
    L = logits.cpu().numpy()
    assert np.isnan(L).any() and np.isinf(L).any()
    ri, rw = oracle.topk_logits(L, k, fn, True)
    np.testing.assert_array_equal(idx.cpu().numpy(), ri)
    fin = np.isfinite(L).all(1)
    np.testing.assert_allclose(w.cpu().numpy()[fin], rw[fin], rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("shape", [(4096, 4096, 128, 8, 0, 8), (2048, 7168, 256, 8, 1, 8),
                                   (3000, 1024, 64, 4, 0, 5), (65536, 1024, 128, 8, 1, 16)])
def test_router_topk_demand(eng, shape):
    """mpb_router_topk_demand: the same routing as mpb_router_topk (bit for
    bit: same kernel, same tile schedule) and demand / demand2 equal to the
    histogram of (source group, selected expert) — what mpb_dispatch_layout
    counts (simulator.cpp:64-80). Covers the cluster tail (decode shape), the
    2-SM pair epilogue (E = 256), E = 64 and a multi-wave batch. A source
    group >= D raises ValidationError at sync."""
    from paper_2604_23150_b200.errors import ValidationError
    T, H, E, k, fn, D = shape
    g = torch.Generator(device="cuda").manual_seed(T + E + D)
    X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    src = torch.randint(0, D, (T,), device="cuda", generator=g).to(torch.uint8)
    src2 = ((torch.arange(T, device="cuda") * 7) % D).to(torch.uint8)
    dem = torch.zeros(D, E, dtype=torch.uint64, device="cuda")
    dem2 = torch.zeros(D, E, dtype=torch.uint64, device="cuda")
    ri, rw = eng.router_topk(X, W, k, fn, True)
    idx, w = eng.router_topk_demand(X, W, k, fn, True, src, D, dem, src2, dem2)
    eng.sync()
    assert torch.equal(idx, ri) and torch.equal(w, rw)
    ih = idx.cpu().numpy().astype(np.int64)
    for s_, d_ in ((src, dem), (src2, dem2)):
        ref = np.zeros((D, E), np.uint64)
        np.add.at(ref, (np.repeat(s_.cpu().numpy().astype(np.int64), k), ih.reshape(-1)), 1)
        np.testing.assert_array_equal(d_.cpu().numpy(), ref)
    bad = src.clone()
    bad[T // 2] = D
    eng.router_topk_demand(X, W, k, fn, True, bad, D, dem)
    with pytest.raises(ValidationError):
        eng.sync()
