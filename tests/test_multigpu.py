"""Real multi-GPU AMSP step (one process per GPU, NVLink peer memory),
bit-exact against the CPU oracle. Needs >= 2 GPUs (gpurun --gpus 2|4)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


CASES = [(2, "2x1", None, "greedy"), (2, "2x1", None, "contiguous"),
         (4, "4x1", None, "greedy"), (4, "2x1", None, "greedy"),
         (4, "2x2", "2x2", "greedy"), (4, "4x1", None, "contiguous")]


@pytest.mark.parametrize("world,os_mesh,dp_mesh,layout", CASES)
def test_torchrun_group(world, os_mesh, dp_mesh, layout):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29531",
           str(REPO / "tests" / "mp_worker.py"), "--os-mesh", os_mesh, "--layout", layout]
    if dp_mesh:
        cmd += ["--dp-mesh", dp_mesh]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO,
                       env={**os.environ, "OMP_NUM_THREADS": "4"})
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(" OK ") == world, out[-4000:]
