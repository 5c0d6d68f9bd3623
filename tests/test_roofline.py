"""B200 step roofline and the roofline-ordered solver (engine/roofline.h,
amsp_step_roofline / amsp_solve_roofline): host-only, no GPU.

- The native per-rank algorithmic bytes equal bench.step_bytes, the
  formulas the bench's roofline fractions are computed with, for every
  candidate plan of several meshes.
- On the measured 27-combo sweep (BASELINE config 5: 1B params, 4 B200s,
  meshes 4x1 / 2x2 / 1x4; profiles/r01_sweep_1b_4gpu_v2.jsonl) the roofline
  solver picks a plan within 1% of the measured best. The reference
  objective (shardplan::solve, kept bit-exact) picks one >= 10% slower.
"""
import json
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402
from paper_2311_00257_b200 import shardplan as S  # noqa: E402
from paper_2311_00257_b200.engine import b200_profile, mesh_group, pshard_layout  # noqa: E402

M = S.DeviceMesh


def _cluster(dp, capacity=180_000_000_000):
    return S.ClusterSpec(dp.per_node, dp.nodes, capacity, dp, S.Topology(dp.nodes, 1, 1.0))


@pytest.mark.parametrize("model,mesh", [("tiny", (2, 1)), ("tiny", (4, 1)), ("tiny", (2, 2)),
                                        ("llama-1b", (4, 1)), ("llama-1b", (1, 4)),
                                        ("tiny", (8, 1)), ("llama-7b", (8, 1))])
def test_step_bytes_match_bench_formulas(model, mesh):
    m = S.model(model)
    tensors = S.model_tensors(m)
    assert tensors == S.llama_tensors(m)
    dp = M(*mesh)
    W = dp.size()
    phi = sum(tensors)
    for plan in S.enumerate_candidates(_cluster(dp)):
        if any(t % plan.sp() for t in tensors):
            continue
        for rank in range(W):
            st, _ = S.step_roofline(tensors, plan, dp, rank)
            # the engine's own k / OS position for this rank
            _, ppos, _ = mesh_group(dp, plan.p, rank)
            _, _, members = mesh_group(dp, plan.os, rank)
            same = [q for q in members if mesh_group(dp, plan.p, q)[1] == ppos]
            _, owned = pshard_layout(tensors, plan.sp(), ppos, len(same), same.index(rank),
                                     "greedy")
            assert st.owned == owned
            hbm, nvl = bench.step_bytes(phi, owned, W, len(same), plan.sp(), plan.sos())
            assert st.hbm_bytes == hbm, (str(plan), rank)
            assert max(st.nvlink_in_bytes, st.nvlink_out_bytes) == nvl, (str(plan), rank)
            assert st.t_step == pytest.approx(max(hbm / S.B200_HBM_BW, nvl / S.B200_NVLINK_BW))
        worst, who = S.step_roofline(tensors, plan, dp)
        assert worst.t_step == max(S.step_roofline(tensors, plan, dp, r)[0].t_step
                                   for r in range(W))
        assert 0 <= who < W


def test_single_rank_has_no_nvlink_and_matches_bench_default():
    m = S.model("llama-7b")
    st, _ = S.step_roofline(m, S.ShardingPlan(), M(1, 1))
    assert st.nvlink_in_bytes == st.nvlink_out_bytes == 0
    assert st.hbm_bytes == 28 * m.total_params  # 188.7 GB: the bench's W=1 roofline
    assert st.t_step == pytest.approx(28 * m.total_params / S.B200_HBM_BW)


def test_roofline_solver_picks_the_measured_best_of_the_sweep():
    rows = [json.loads(line) for line in
            (REPO / "profiles" / "r01_sweep_1b_4gpu_v2.jsonl").read_text().splitlines()]
    model = S.model("llama-1b", seq_len=4096)
    for res in rows:
        a, b = map(int, res["mesh"].split("x"))
        dp = M(a, b)
        # the sweep's planner input: the measured NCCL profile (tools/profile_nvlink.py)
        prof = S.BandwidthProfile.load(str(REPO / res["profile"]))
        ranked = S.solve_roofline(model, _cluster(dp), prof)
        pick = str(ranked[0][0].plan)
        measured = {r["plan"]: r for r in res["rows"] if "pipeline_ms" in r}
        best_pipe = min(r["pipeline_ms"] for r in measured.values())
        best_over = min(r["overlap_step_ms"] for r in measured.values())
        assert measured[pick]["pipeline_ms"] <= 1.01 * best_pipe, (res["mesh"], pick)
        assert measured[pick]["overlap_step_ms"] <= 1.01 * best_over, (res["mesh"], pick)
        # the reference objective's pick (communication time only) on the same cluster
        ref_pick = str(S.solve(model, _cluster(dp), prof).best.plan)
        assert ref_pick == res["solver_pick"]
        assert measured[ref_pick]["pipeline_ms"] >= 1.5 * best_pipe
        assert measured[ref_pick]["overlap_step_ms"] >= 1.1 * best_over
        # every measured (valid) plan is ranked, roofline-ordered
        ts = [st.t_step for _, st in ranked]
        assert ts == sorted(ts)
        assert set(measured) <= {str(r.plan) for r, _ in ranked}


def test_roofline_solver_reports_infeasible_with_the_leanest_plan():
    model = S.model("llama-7b")
    with pytest.raises(S.NoFeasiblePlanError) as ei:
        S.solve_roofline(model, _cluster(M(2, 1), capacity=10_000_000_000), b200_profile())
    assert ei.value.closest().plan == S.ShardingPlan(M(2, 1), M(2, 1), M(2, 1))


@pytest.mark.parametrize("s2", [2, 4])
def test_zeropp_secondary_mesh_bytes(s2):
    """ZeRO++ (plan.secondary_params): the backward all-gather pass moves
    2*Phi*(s2-1)/s2 per direction over the secondary group instead of
    2*Phi*(s_p-1)/s_p, and the forward pass refreshes the Phi/s2 slice; the
    native roofline and bench.step_bytes agree."""
    m = S.model("llama-13b")
    tensors = S.model_tensors(m)
    phi = sum(tensors)
    dp = M(8, 1)
    plan = S.ShardingPlan(M(8, 1), M(8, 1), M(8, 1), secondary_params=M(s2, 1))
    st, _ = S.step_roofline(tensors, plan, dp, 0)
    _, owned = pshard_layout(tensors, 8, 0, 1, 0, "greedy")
    hbm, nvl = bench.step_bytes(phi, owned, 8, 1, 8, 8, s2=s2)
    assert (st.hbm_bytes, max(st.nvlink_in_bytes, st.nvlink_out_bytes)) == (hbm, nvl)
    plain, _ = S.step_roofline(tensors, S.ShardingPlan(M(8, 1), M(8, 1), M(8, 1)), dp, 0)
    fewer = 2 * phi * 7 // 8 - 2 * phi * (s2 - 1) // s2
    assert max(plain.nvlink_in_bytes, plain.nvlink_out_bytes) - nvl == fewer


def test_roofline_solver_ranks_zeropp_variants():
    """The roofline solver also ranks the ZeRO++ variant (secondary mesh
    strictly inside P) of every parameter-sharded candidate; on 13B / 4 GPUs
    it moves fewer NVLink bytes than plain ZeRO-3 and ranks above it."""
    m = S.model("llama-13b")
    ranked = S.solve_roofline(m, _cluster(M(4, 1)), b200_profile())
    plans = [str(r[0].plan) for r in ranked]
    zpp, z3 = "p=4x1,g=4x1,os=4x1,p2=2x1", "p=4x1,g=4x1,os=4x1"
    assert zpp in plans and z3 in plans
    assert plans.index(zpp) < plans.index(z3)
    # the reference objective (solve) is unchanged: no secondary candidates
    assert all(r.plan.secondary_params is None
               for r in S.solve(m, _cluster(M(4, 1)), b200_profile(),
                                keep_all_results=True).all_results)
