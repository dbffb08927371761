"""CPU: the reference's own unit suites (132 doctest cases, via the shim in
oracle/doctest_shim) and acceptance criteria, built UNMODIFIED from
/root/reference sources by oracle/Makefile, pass against the reference core —
the checker this repo's oracle is pinned to."""
import subprocess

import pytest

from tests.conftest import ROOT

REF = ROOT / "oracle" / "_ref"


@pytest.mark.parametrize("binary", ["ref_unit_tests", "ref_acceptance"])
def test_reference_suite_passes(binary):
    exe = REF / binary
    if not exe.exists():
        pytest.skip(f"{exe} not built (make -C oracle ref needs /root/reference)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600, cwd="/tmp")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    if binary == "ref_unit_tests":
        assert "test cases: 132 | passed: 132 | failed: 0" in r.stdout
    else:
        assert "all 9 criteria passed" in r.stdout
