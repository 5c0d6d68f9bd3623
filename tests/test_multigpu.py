"""Real multi-process AMSP step (one process per rank, cudaIpc peer memory,
device-side cross-GPU barriers), bit-exact against the CPU oracle.

With >= W GPUs every rank has its own B200 (NVLink). With fewer GPUs the
ranks could share devices ("oversubscribed"): the code path is identical --
cudaIpc handles, the barrier_kernel flag protocol, the __threadfence_system
release of peer stores, the host step's per-chunk barriers -- only the
timing is meaningless. But ranks that spin on one another's flags, run as
processes on ONE GPU, have raised Xid 109 (context-switch timeout) on B200
with driver 580.159 (B200_PROFILING.md, "Do not run kernels that wait on one
another ... as separate launches on one GPU"), which leaves the GPU unusable.
So oversubscribed groups only run when AMSP_OVERSUB=1 is set explicitly;
otherwise a case needs one GPU per rank. The single-GPU driver run covers
the barrier protocol in one process instead (tests/test_engine_gpu.py,
emulated groups with real barrier kernels on per-rank streams)."""
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


CASES = [(2, "2x1", None, "greedy", None), (2, "2x1", None, "contiguous", None),
         (2, "2x1", None, "greedy", "2x1"),                      # ZeRO-3
         (4, "4x1", None, "greedy", None), (4, "2x1", None, "greedy", None),
         (4, "2x2", "2x2", "greedy", None), (4, "4x1", None, "contiguous", None),
         (4, "4x1", None, "greedy", "4x1"),                      # ZeRO-3
         (4, "4x1", None, "greedy", "2x1"),                      # AMSP-13B-style
         (2, "2x1", None, "greedy", "sched"), (4, "4x1", None, "greedy", "sched"),
         (4, "4x1", None, "greedy", "4x1+sched"), (4, "2x1", None, "greedy", "sched")]
CASES = [c + (0,) for c in CASES] + [
    # auto (0) is the TMA bulk-copy pipeline (variant 5) for aligned layouts;
    # variant 6 = the deeper 1-CTA/SM ring, 1 / 2 = the LDG kernels
    (2, "2x1", None, "greedy", None, 6), (4, "4x1", None, "greedy", None, 6),
    (2, "2x1", None, "greedy", None, 2), (4, "4x1", None, "greedy", None, 1),
    (4, "2x1", None, "greedy", None, 2),
    # host-buffer step: chunked H2D pipelined with per-chunk barriers
    (2, "2x1", None, "greedy", "host", 0), (4, "4x1", None, "greedy", "host", 0),
    (4, "2x1", None, "greedy", "host", 0),
    # ZeRO-3 all-gathers by the TMA bulk-copy kernel, in the step and in the scheduler
    (4, "4x1", None, "greedy", "4x1+tma", 0), (4, "4x1", None, "greedy", "4x1+sched+tma", 0),
    # W=8 (the BASELINE 8xB200 meshes) with several ranks per GPU: ZeRO-1, ZeRO-1
    # on the 2x4 virtual-node mesh, ZeRO-3, AMSP-13B (p=4, os=8)
    (8, "8x1", None, "greedy", "oversub", 0), (8, "2x4", "2x4", "greedy", "oversub", 0),
    (8, "8x1", None, "greedy", "8x1+oversub", 0), (8, "8x1", None, "greedy", "4x1+oversub", 0),
    (8, "8x1", None, "greedy", "sched+oversub", 0), (8, "4x1", None, "greedy", "oversub", 2),
    # fused kernel with bulk-store drains (variants 7 / 8)
    (2, "2x1", None, "greedy", None, 7), (4, "4x1", None, "greedy", None, 7),
    (4, "2x1", None, "greedy", None, 8),
    # ring-depth variants (W=2 default 11, W=4 default 10) forced on other groups
    (4, "4x1", None, "greedy", None, 11), (2, "2x1", None, "greedy", None, 10),
    # scheduler with copy-engine staged gradient reduces
    (2, "2x1", None, "greedy", "sched+dmared", 0), (4, "4x1", None, "greedy", "sched+dmared", 0),
    (4, "4x1", None, "greedy", "4x1+sched+tma+dmared", 0),
    (4, "2x1", None, "greedy", "sched+dmared", 0),
    # M > 1 micro-batches with gradient sharding: the
    # pipeline API (accumulate per micro-batch, step on the last) ...
    (2, "2x1", None, "greedy", "g=2x1+mb=2", 0),             # ZeRO-2
    (4, "4x1", None, "greedy", "4x1+mb=2", 0),               # ZeRO-3
    (4, "4x1", None, "greedy", "2x1+mb=3", 0),               # s_g = s_p = 2 < s_os
    (4, "2x1", None, "greedy", "g=2x1+mb=2", 0),             # g = os = 2, two replicas
    (4, "4x1", None, "greedy", "mb=3", 0),                   # ZeRO-1, in place
    (8, "2x4", "2x4", "greedy", "g=2x4+mb=2+oversub", 0),    # BASELINE partial 2x4
    # ... and the overlap scheduler, gradients written by the grad-weight
    # events during the step (no host barriers at all)
    (2, "2x1", None, "greedy", "g=2x1+mb=2+sched+synth", 0),
    (4, "4x1", None, "greedy", "4x1+mb=2+sched+synth", 0),
    (4, "4x1", None, "greedy", "2x1+mb=2+sched+synth", 0),
    (4, "2x2", "2x2", "greedy", "g=2x2+mb=2+sched+synth", 0),
    (4, "4x1", None, "greedy", "mb=2+sched+synth", 0),
    (4, "2x1", None, "greedy", "g=2x1+mb=3+sched+synth", 0),
    # two schedulers on one engine, alternating steps, no host sync (the
    # barrier epochs must keep growing across schedulers)
    (2, "2x1", None, "greedy", "sched+synth+two", 0),
    (4, "4x1", None, "greedy", "4x1+sched+synth+two", 0),
    # the gradient ring at the schedule's smallest size (D_g = G shard + ring)
    (2, "2x1", None, "greedy", "g=2x1+sched+synth+ring", 0),
    (2, "2x1", None, "greedy", "g=2x1+mb=3+sched+synth+ring", 0),
    (4, "4x1", None, "greedy", "4x1+mb=2+sched+synth+ring", 0),
    (4, "4x1", None, "greedy", "2x1+mb=2+sched+synth+ring", 0),
    (4, "2x2", "2x2", "greedy", "g=2x2+mb=2+sched+synth+ring", 0),
    # ZeRO++ secondary parameter mesh (backward all-gathers from the secondary group)
    (4, "4x1", None, "greedy", "4x1+p2=2x1", 0),
    (4, "4x1", None, "greedy", "4x1+p2=2x1+push", 0),
    (4, "4x1", None, "greedy", "4x1+push", 0),
    (2, "2x1", None, "greedy", "2x1+push", 0),
    (4, "4x1", None, "greedy", "4x1+p2=2x1+sched+synth", 0),
    (4, "4x1", None, "greedy", "4x1+p2=2x1+mb=2+sched+synth", 0)]

# With AMSP_OVERSUB=1: run on a 1-GPU box with all ranks sharing the device.
CORE = {(2, "2x1", None, "greedy", None, 0), (2, "2x1", None, "greedy", "2x1", 0),
        (2, "2x1", None, "greedy", "host", 0), (4, "2x2", "2x2", "greedy", None, 0),
        (2, "2x1", None, "greedy", "sched", 0), (8, "8x1", None, "greedy", "oversub", 0),
        (2, "2x1", None, "greedy", "g=2x1+mb=2", 0), (4, "4x1", None, "greedy", "4x1+mb=2", 0),
        (8, "2x4", "2x4", "greedy", "g=2x4+mb=2+oversub", 0),
        (2, "2x1", None, "greedy", "g=2x1+mb=2+sched+synth", 0),
        (4, "4x1", None, "greedy", "4x1+mb=2+sched+synth", 0),
        (2, "2x1", None, "greedy", "sched+synth+two", 0)}


@pytest.mark.parametrize("world,os_mesh,dp_mesh,layout,p_mesh,variant", CASES)
def test_torchrun_group(world, os_mesh, dp_mesh, layout, p_mesh, variant):
    # p_mesh: "[AxB][+sched][+tma]" or "sched" / "host"
    case = (world, os_mesh, dp_mesh, layout, p_mesh, variant)
    words = (p_mesh or "").split("+")
    host, sched, tma = "host" in words, "sched" in words, "tma" in words
    meshes = [w for w in words if "x" in w and "=" not in w]
    p_mesh = meshes[0] if meshes else None
    opts = dict(w.split("=") for w in words if "=" in w)
    need = world
    if os.environ.get("AMSP_OVERSUB") == "1":
        need = 1 if case in CORE else 2 if "oversub" in words else world
    if _ngpus() < need:
        pytest.skip(f"needs {need} GPUs (oversubscribed groups only with AMSP_OVERSUB=1)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29531",
           str(REPO / "tests" / "mp_worker.py"), "--os-mesh", os_mesh, "--layout", layout]
    if dp_mesh:
        cmd += ["--dp-mesh", dp_mesh]
    if p_mesh:
        cmd += ["--p-mesh", p_mesh]
    if sched:
        cmd += ["--sched"]
    if variant:
        cmd += ["--variant", str(variant)]
    if host:
        cmd += ["--host", "--model", "chunky", "--steps", "2"]
    if tma:
        cmd += ["--gather", "tma"]
    if "push" in words:
        cmd += ["--gather", "push"]
    if "dmared" in words:
        cmd += ["--reduce", "dma"]
    if "g" in opts:
        cmd += ["--g-mesh", opts["g"]]
    if "mb" in opts:
        cmd += ["--micro-batches", opts["mb"]]
    if "synth" in words:
        cmd += ["--synth"]
    if "two" in words:
        cmd += ["--two-scheds"]
    if "ring" in words:
        cmd += ["--ring"]
    if "p2" in opts:
        cmd += ["--p2-mesh", opts["p2"]]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO,
                       env={**os.environ, "OMP_NUM_THREADS": "4"})
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(" OK ") == world, out[-4000:]


# Every element at the BASELINE model sizes (streamed oracle, tests/fullcheck.py):
# LLaMA-7B ZeRO-1 at W=2 and W=4, 7B on the 2x2 virtual-node mesh, 13B ZeRO-3 at W=4.
FULL = [(2, "llama-7b", "2x1", None, None), (4, "llama-7b", "4x1", None, None),
        (4, "llama-7b", "2x2", "2x2", None), (4, "llama-13b", "4x1", None, "4x1")]


@pytest.mark.parametrize("world,model,os_mesh,dp_mesh,p_mesh", FULL)
def test_torchrun_fullsize_every_element(world, model, os_mesh, dp_mesh, p_mesh):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29532",
           str(REPO / "tests" / "mp_worker.py"), "--os-mesh", os_mesh, "--model", model,
           "--steps", "2", "--full"]
    if dp_mesh:
        cmd += ["--dp-mesh", dp_mesh]
    if p_mesh:
        cmd += ["--p-mesh", p_mesh]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=REPO)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(" OK full-size") == world, out[-4000:]
