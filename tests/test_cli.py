"""CLI: commands, exit codes 0/1/2, deterministic reports,
profile import round trip."""
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]


def run(*args, cwd=REPO):
    r = subprocess.run([sys.executable, "-m", "paper_2311_00257_b200.cli", *args],
                       capture_output=True, text=True, cwd=cwd)
    return r.returncode, r.stdout, r.stderr


def cfg(tmp_path, **over):
    c = {"model": {"llama": "llama-7b"},
         "cluster": {"gpus_per_node": 8, "node_count": 1, "gpu_memory_capacity": 80e9,
                     "dp_mesh": [8, 1]}}
    c.update(over)
    p = tmp_path / "run.json"
    p.write_text(json.dumps(c))
    return str(p)


def test_plan_report_deterministic(tmp_path):
    c = cfg(tmp_path)
    rc1, out1, _ = run("plan", "--config", c, "--all-candidates")
    rc2, out2, _ = run("plan", "--config", c, "--all-candidates")
    assert rc1 == rc2 == 0 and out1 == out2
    rep = json.loads(out1)
    assert rep["candidates_evaluated"] == 16 and len(rep["all_candidates"]) == 16
    assert rep["config"]["model"] == {"llama": "llama-7b"}


def test_plan_infeasible_exit_2(tmp_path):
    c = cfg(tmp_path, cluster={"gpus_per_node": 8, "node_count": 1, "gpu_memory_capacity": 1,
                               "dp_mesh": [8, 1]})
    rc, out, _ = run("plan", "--config", c)
    assert rc == 2
    rep = json.loads(out)
    assert rep["feasible"] is False and rep["closest"]["plan"] == "p=8x1,g=8x1,os=8x1"


def test_config_errors_exit_1(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"model": {"llama": "llama-7b"}, "cluster": {"gpus": 8}}')
    rc, _, err = run("plan", "--config", str(bad))
    assert rc == 1 and "config.cluster.gpus" in err
    bad.write_text("{not json")
    rc, _, err = run("plan", "--config", str(bad))
    assert rc == 1 and "config" in err
    rc, _, err = run("simulate", "--config", cfg(tmp_path), "--plan", "p=1x1,g=4x1,os=8x1")
    assert rc == 1 and "s_g in {s_p, s_os}" in err


def test_simulate_tiers_monotone_and_trace(tmp_path):
    c = cfg(tmp_path)
    steps = []
    for tier in ("none", "ag_rs", "ag_rs_ar", "ag_rs_ar_bc"):
        rc, out, _ = run("simulate", "--config", c, "--preset", "ZeRO-3", "--overlap", tier)
        assert rc == 0
        steps.append(json.loads(out)["step_time"])
    assert steps == sorted(steps, reverse=True)
    tr = tmp_path / "t.json"
    rc, _, _ = run("simulate", "--config", c, "--preset", "ZeRO-1", "--trace", str(tr))
    assert rc == 0 and json.loads(tr.read_text())[0]["ph"] == "X"


def test_compare_keeps_infeasible_rows(tmp_path):
    rc, out, _ = run("compare", "--config", cfg(tmp_path))
    assert rc == 0
    rows = json.loads(out)["rows"]
    names = [r["name"] for r in rows]
    assert set(names) == {"ZeRO-1", "ZeRO-3", "MiCS", "ZeRO++", "AMSP-7B", "AMSP-13B",
                          "AMSP-30B", "solver"}
    assert "error" in next(r for r in rows if r["name"] == "AMSP-30B")


def test_import_profile_roundtrip(tmp_path):
    csv = tmp_path / "p.csv"
    csv.write_text("op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\n"
                   "allreduce,4096,8,1,2e9\nallreduce,1024,8,1,1e9\n")
    out = tmp_path / "p.json"
    assert run("import-profile", str(csv), str(out))[0] == 0
    first = out.read_text()
    assert json.loads(first) == {"allreduce/8 x 1": [[1024, 1e9], [4096, 2e9]]}
    csv.write_text("op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\n"
                   "allreduce,1,8,1,1\nallreduce,1,8,1,2\n")
    rc, _, err = run("import-profile", str(csv), str(out))
    assert rc == 1 and "duplicate key" in err
    # measured profile feeds the planner
    rc, out2, _ = run("plan", "--config", cfg(tmp_path, profile_path=str(REPO / "profiles" /
                                                                          "b200_nccl_4gpu.csv"),
                                              cluster={"gpus_per_node": 4, "node_count": 1,
                                                       "gpu_memory_capacity": 180e9,
                                                       "dp_mesh": [4, 1]}))
    assert rc == 0 and json.loads(out2)["best"]["plan"]


def test_plan_roofline_objective(tmp_path):
    """`plan --objective roofline` ranks the same candidates by the B200 step
    roofline: on 8 B200s (180 GB) it picks a plan that shards the optimizer
    state over all 8 GPUs, where the reference objective keeps the replica."""
    c = cfg(tmp_path, cluster={"gpus_per_node": 8, "node_count": 1,
                               "gpu_memory_capacity": 180e9, "dp_mesh": [8, 1]})
    rc, out, _ = run("plan", "--config", c, "--objective", "roofline", "--all-candidates")
    assert rc == 0
    rep = json.loads(out)
    assert rep["objective"]["name"] == "roofline"
    best = rep["best"]
    assert best["plan"].endswith("os=8x1") and best["plan"].startswith("p=1x1")
    steps = [r["step_roofline"]["t_step"] for r in rep["all_candidates"]]
    assert steps == sorted(steps) and best["step_roofline"]["t_step"] == steps[0]
    rc, out, _ = run("plan", "--config", c)
    assert rc == 0 and json.loads(out)["best"]["plan"] != best["plan"]


def test_roofline_command_projects_the_8_gpu_configs(tmp_path):
    """`roofline` on the BASELINE 8xB200 configs: 7B ZeRO-1 and the partial
    plan (G/OS over the 2x4 mesh) move identical bytes (23.7 GB/dir NVLink,
    bound 30.8 ms); 13B ZeRO-3 is bound by 68.3 GB/dir."""
    c = cfg(tmp_path, cluster={"gpus_per_node": 8, "node_count": 1,
                               "gpu_memory_capacity": 180e9, "dp_mesh": [8, 1]})
    rc, out, _ = run("roofline", "--config", c, "--plan", "p=1x1,g=1x1,os=8x1")
    assert rc == 0
    z1 = json.loads(out)
    assert len(z1["ranks"]) == 8 and z1["params"] == 6738415616
    assert abs(z1["step"]["t_step"] - 0.03076) < 1e-4
    assert z1["step"]["nvlink_in_bytes"] == max(r["nvlink_in_bytes"] for r in z1["ranks"])
    c2 = cfg(tmp_path, cluster={"gpus_per_node": 2, "node_count": 4,
                                "gpu_memory_capacity": 180e9, "dp_mesh": [2, 4]})
    rc, out, _ = run("roofline", "--config", c2, "--plan", "p=1x1,g=2x4,os=2x4")
    assert rc == 0 and json.loads(out)["step"]["t_step"] == z1["step"]["t_step"]
    c3 = cfg(tmp_path, model={"llama": "llama-13b"},
             cluster={"gpus_per_node": 8, "node_count": 1, "gpu_memory_capacity": 180e9,
                      "dp_mesh": [8, 1]})
    rc, out, _ = run("roofline", "--config", c3, "--preset", "ZeRO-3")
    z3 = json.loads(out)
    assert rc == 0 and z3["plan"] == "p=8x1,g=8x1,os=8x1"
    assert z3["step"]["nvlink_in_bytes"] == 68333287680
    rc, _, err = run("roofline", "--config", c, "--plan", "p=1x1,g=4x1,os=8x1")
    assert rc == 1 and "violates" in err
