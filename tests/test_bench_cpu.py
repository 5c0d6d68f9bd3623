"""bench.py's reference arm runs on host cores only, so its JSON contract is
checked here on CPU: one line with the shared metric / unit / config keys,
`impl: reference`, a cpu_baseline and an e2e object; under torchrun only
rank 0 prints and every rank exits 0."""
import json
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
        "cpu_baseline", "e2e", "impl"}


def _lines(out: str):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _check(line, world):
    assert KEYS <= set(line), KEYS - set(line)
    assert line["impl"] == "reference" and line["n_gpus"] == world
    assert line["value"] > 0 and line["unit"] == "params/s" and line["higher_is_better"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["model"] == "llama-7b" and line["config"]["parallelism"] == f"dp{world}"
    # the step is measured on the bounded sample, so steps x ms_per_step is real time
    assert line["ms_per_step"] < line["ms_per_step_full_workload_extrapolated"]
    planner = line["planner"]
    if isinstance(planner, list):  # oracle/_ref built (the reference is mounted here)
        entries = {p["entry"] for p in planner}
        assert entries == {"solve", "build_schedule+simulate_step"}
        assert all(p["best_us"] > 0 for p in planner)


def test_reference_arm_single_process():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], cwd=REPO, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    _check(lines[0], 1)


def test_reference_arm_under_torchrun_rank0_only():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29641", "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=300,
                       env={**os.environ, "OMP_NUM_THREADS": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    _check(lines[0], 2)


def test_reference_arm_reports_the_roofline_solver_plan():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--gpus", "1", "--mesh", "4x1", "--plan", "roofline"],
                       cwd=REPO, capture_output=True, text=True, timeout=300,
                       env={**os.environ, "WORLD_SIZE": "1"})
    # --mesh 4x1 with one process: the plan is still resolved for the 4-GPU mesh
    assert r.returncode == 0, r.stderr[-2000:]
    line = _lines(r.stdout)[0]
    assert line["config"]["plan"] == "p=1x1,g=1x1,os=4x1"
    assert line["config"]["dp_mesh"] == "4x1"


def test_step_bytes_phases_and_micro_batches():
    """bench.step_bytes: ZeRO-1 moves 4*Phi*(W-1)/W per direction;
    the phase split sums to the totals; M > 1 with s_g > 1 adds (M-1)
    accumulation passes; s_p > 1 adds the two all-gather passes."""
    sys.path.insert(0, str(REPO))
    import bench
    phi, W = 6_738_415_616, 4
    hbm, nvl = bench.step_bytes(phi, phi // W, W, W)
    assert abs(nvl - 4 * phi * (W - 1) / W) <= 8
    assert hbm == 24 * (phi // W) + 2 * phi + 2 * phi
    for kw in ({"micro": 4, "acc_elems": phi // 2, "sg": 2, "sos": 2},
               {"sp": 4, "sos": 4}, {}):
        k = 2 if kw.get("sos") == 2 else (1 if kw.get("sp") == 4 else W)
        owned = phi // kw.get("sos", W)
        phases = bench.step_bytes(phi, owned, W, k, phases=True, **kw)
        tot = bench.step_bytes(phi, owned, W, k, **kw)
        assert (sum(p[1] for p in phases), sum(p[2] for p in phases)) == tot
    acc = bench.step_bytes(phi, phi // 2, W, 2, sos=2, micro=4, acc_elems=phi // 2, sg=2,
                           phases=True)
    assert [p[0] for p in acc] == ["accumulate", "update"]
    # 3 accumulations: each pulls the (s_g-1)/s_g remote half of the G block
    assert acc[0][2] == 3 * 2 * (phi // 2) * 1
    z3 = bench.step_bytes(13_015_864_320, 13_015_864_320 // 4, 4, 1, sp=4, sos=4, phases=True)
    assert [p[0] for p in z3] == ["all_gather", "update"]
