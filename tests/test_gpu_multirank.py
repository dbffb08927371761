"""GPU, N>1: the fused NVLink dispatch / combine (K6-P2P) and the NCCL
all-to-all-v path across real ranks (tools/a2a_check.py under torchrun): the
rows each rank receives, the count matrix and the combined output are bit-exact
against an all-gathered restatement and the world-1 local permute. Skips on a
one-GPU box."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("world", [2, 4])
def test_k6_multirank_bit_identity(world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        f"--master-port={29600 + world}", str(ROOT / "tools" / "a2a_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["all_ranks_ok"], res
    assert res["rank0"]["recv_rows"] > 0


@pytest.mark.parametrize("world", [2, 4])
def test_step_nccl_in_plan_equals_torch_collectives(world):
    """The C++ step's own NCCL collectives (inside its CUDA graph) produce the
    same statistics and LayerSim tables as torch.distributed collectives
    between the phases, bit for bit, on every rank (tools/step_nccl_check.py)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        f"--master-port={29640 + world}",
                        str(ROOT / "tools" / "step_nccl_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    assert json.loads(lines[-1])["all_ranks_bit_identical"]
