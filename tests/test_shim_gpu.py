"""GPU: the reference's UNMODIFIED unit suites (132 cases), acceptance
criteria and run_pipeline, linked with the C++ drop-in
(paper_2604_23150_b200/shim: simulator_b200, trace_b200, metrics_b200,
clustering_b200, placement_b200) in place of the reference's simulator.cpp,
trace.cpp, metrics.cpp, clustering.cpp and placement.cpp, so every hot-path
call they make — parsing, matrix builds, statistics, k-means, placements,
simulate_layer / compare_strategies — runs through the C ABI on the B200. Binaries are built here by
`make -C paper_2604_23150_b200/shim tests` (needs /root/reference) and travel
to the GPU box prebuilt."""
import subprocess

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu
BUILD = ROOT / "paper_2604_23150_b200" / "shim" / "build"


@pytest.mark.parametrize("binary", ["shim_unit_tests", "shim_acceptance"])
def test_reference_suites_through_b200_shim(binary):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = BUILD / binary
    if not exe.exists():
        pytest.skip(f"{exe} not built (make -C paper_2604_23150_b200/shim tests)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, cwd="/tmp")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    if binary == "shim_unit_tests":
        assert "test cases: 132 | passed: 132 | failed: 0" in r.stdout
    else:
        assert "all 9 criteria passed" in r.stdout


@pytest.mark.parametrize("config", ["dsv3_c2", "qwen3_c1", "desk_default"])
def test_run_pipeline_byte_identical(tmp_path, config):
    """The reference's own run_pipeline (pipeline.cpp:316-443, unmodified)
    linked against the B200 drop-in (all five hot-path TUs swapped) writes
    the same artifacts, byte for byte, as when linked against the reference's
    CPU core: trace.jsonl, imbalance / correlation CSVs, cluster report and
    model, placements, simulation CSVs, classification, summary, manifest."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    shim = BUILD / "shim_pipeline"
    ref = ROOT / "oracle" / "_ref" / "ref_pipeline"
    if not shim.exists() or not ref.exists():
        pytest.skip("pipeline binaries not built (make -C oracle ref; make -C .../shim tests)")
    cfg = ROOT / "configs" / f"{config}.json"
    outs = {}
    for name, exe in (("shim", shim), ("ref", ref)):
        out = tmp_path / name
        r = subprocess.run([str(exe), str(cfg), str(out)], capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[name] = out
    files = sorted(p.name for p in outs["ref"].iterdir() if p.is_file())
    assert files == sorted(p.name for p in outs["shim"].iterdir() if p.is_file())
    assert "simulation.csv" in files and "trace.jsonl" in files
    for f in files:
        if f.endswith(".lock"):
            continue
        assert (outs["shim"] / f).read_bytes() == (outs["ref"] / f).read_bytes(), f
