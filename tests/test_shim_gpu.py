"""GPU: the reference's UNMODIFIED unit suites (132 cases) and acceptance
criteria, linked with paper_2604_23150_b200/shim/simulator_b200.cpp in place
of the reference's simulator.cpp, so every simulate_layer / compare_strategies
call they make runs on the B200 through the C ABI. Binaries are built here by
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
