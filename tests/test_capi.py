"""C-ABI boundary (include/amsp_c.h): the library loads without a GPU,
exports every declared symbol, and the planner half reproduces the SPEC's
known-answer examples and acceptance properties through the
Python mirror of the reference API."""
import math
import random
import re
from pathlib import Path

import pytest

from paper_2311_00257_b200 import _native as N
from paper_2311_00257_b200 import shardplan as S

REPO = Path(__file__).resolve().parents[1]
M = S.DeviceMesh


def test_every_declared_symbol_is_exported():
    header = (REPO / "include" / "amsp_c.h").read_text()
    declared = set(re.findall(r"\b(amsp_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 39
    lib = N.lib()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(N.SIGNATURES) <= declared


def test_known_answers_spec_appendix():
    # SPEC.md:136 ring AR 1024 B, p=4, alpha=0, w=1e9
    assert S.ring_time("allreduce", 1024, 4, 0.0, 1e9) == pytest.approx(1.536e-6, rel=1e-15)
    # interpolation: 2 MiB between (1 MiB, 50e9) and (4 MiB, 80e9) -> 65e9
    csv = ("op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\n"
           "allreduce,1048576,8,2,50e9\nallreduce,4194304,8,2,80e9\n")
    prof = S.BandwidthProfile.from_csv(csv)
    assert prof.collective_time("allreduce", 2 << 20, M(8, 2)) == pytest.approx(
        (2 << 20) / 65e9, rel=1e-15)
    # memory exactness (acceptance 1)
    m = S.ModelSpec(7_000_000_000, 32, 1, [200_000_000], 4096, 4096, 1, 1, 32000)
    assert S.memory_breakdown(m, S.ShardingPlan()).d_modelstate == 112e9
    full = S.ShardingPlan(M(8, 128), M(8, 128), M(8, 128))
    assert S.memory_breakdown(m, full).d_modelstate == 112e9 / 1024
    # greedy [7,5,4,3,1] k=2
    assert S.partition_tensors_greedy([7, 5, 4, 3, 1], 2) == ([0, 1, 1, 0, 1], [10, 10])


def test_ring_identity_acceptance_2():
    rng = random.Random(7)
    for _ in range(1000):
        v, p = rng.uniform(0, 1e10), rng.randint(1, 1024)
        a, w = rng.uniform(0, 1e-4), rng.uniform(1e8, 1e12)
        ar = S.ring_time("allreduce", v, p, a, w)
        rs = S.ring_time("reducescatter", v, p, a, w)
        ag = S.ring_time("allgather", v, p, a, w)
        assert math.isclose(ar, rs + ag, rel_tol=1e-12, abs_tol=0.0) or ar == rs + ag


def _profile():
    meshes = [M(a, b) for a in range(1, 9) for b in (1, 2, 4, 8)]
    return S.BandwidthProfile.synthetic((5e-6, 770e9), (10e-6, 50e9), meshes,
                                        [1 << k for k in range(10, 35, 2)])


def test_solver_table_iii_and_infeasible():
    prof = _profile()
    m7 = S.model("llama-7b")
    c = S.ClusterSpec(8, 1, 80_000_000_000, M(8, 1))
    rep = S.solve(m7, c, prof, keep_all_results=True)
    assert rep.candidates_evaluated == 16 and rep.candidates_filtered == 512 - 16
    ranks = sorted(r.rank for r in rep.all_results)
    assert ranks == list(range(16))
    assert S.validate_plan(rep.best.plan, c).ok()
    tiny_cap = S.ClusterSpec(8, 1, 1000, M(8, 1))
    with pytest.raises(S.NoFeasiblePlanError) as ei:
        S.solve(m7, tiny_cap, prof)
    assert ei.value.closest().plan == S.ShardingPlan(M(8, 1), M(8, 1), M(8, 1))
    assert "no feasible plan" in str(ei.value)


def test_enumerate_equals_filtered_grid_acceptance_4():
    for R in range(1, 5):
        for N_ in range(1, 4):
            c = S.ClusterSpec(R, N_, 1 << 40, M(R, N_), S.Topology(N_, 1, 1.0))
            cands = {p.lex_key() for p in S.enumerate_candidates(c)}
            grid = set()
            axes = [(a, b) for a in range(1, R + 1) for b in range(1, N_ + 1)]
            for p in axes:
                for g in axes:
                    for o in axes:
                        plan = S.ShardingPlan(M(*p), M(*g), M(*o))
                        if S.validate_plan(plan, c).ok():
                            grid.add(plan.lex_key())
            assert cands == grid, (R, N_)


def test_sim_closed_form_and_tier_monotone():
    prof = _profile()
    m = S.model("tiny")
    c = S.ClusterSpec(4, 1, 1 << 40, M(4, 1))
    for plan in S.enumerate_candidates(c):
        times = [S.simulate(m, c, plan, prof, sim=S.SimConfig(overlap_tier=t)).step_time
                 for t in S.SimConfig.TIERS]
        assert times == sorted(times, reverse=True), (str(plan), times)
        # tier none telescopes to compute + T_comm (acceptance 5)
        comm = S.total_comm_time(m, c, plan, prof).total
        zero = S.simulate(m, c, plan, prof, sim=S.SimConfig(overlap_tier="none",
                                                              peak_flops_per_gpu=1e30))
        assert zero.step_time == pytest.approx(comm, rel=1e-9, abs=1e-15)


def test_trace_schema():
    prof = _profile()
    m = S.model("tiny")
    c = S.ClusterSpec(2, 1, 1 << 40, M(2, 1))
    r = S.simulate(m, c, S.preset("ZeRO-3", c), prof, with_trace=True)
    import json
    events = json.loads(r.trace)
    assert len(events) == r.n_events
    assert {"name", "ph", "ts", "dur", "pid", "tid"} == set(events[0])


def test_error_codes():
    c = S.ClusterSpec(8, 1, 0, M(8, 1))  # capacity 0 -> Error (code 1)
    with pytest.raises(N.InvalidConfig, match="gpu_memory_capacity"):
        S.enumerate_candidates(c)
    with pytest.raises(N.InvalidConfig, match="unknown preset"):
        S.preset("ZeRO-2", S.ClusterSpec(8, 1, 1, M(8, 1)))
    with pytest.raises(N.InvalidConfig, match="duplicate key"):
        S.BandwidthProfile.from_csv("op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\n"
                                    "allreduce,1,2,1,1\nallreduce,1,2,1,2\n")


def test_profile_roundtrip_byte_stable():
    prof = _profile()
    j = prof.to_canonical_json()
    assert S.BandwidthProfile.from_json(j).to_canonical_json() == j
