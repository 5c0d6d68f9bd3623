"""Command-line front end of the planner.

  python -m paper_2311_00257_b200.cli plan      --config run.json [--profile p.csv|.json]
                                                [--out report.json] [--all-candidates] [--pretty]
  python -m paper_2311_00257_b200.cli simulate  --config run.json [--preset NAME | --plan SPEC]
                                                [--overlap TIER] [--trace trace.json]
  python -m paper_2311_00257_b200.cli compare   --config run.json
  python -m paper_2311_00257_b200.cli roofline  --config run.json [--preset NAME | --plan SPEC]
  python -m paper_2311_00257_b200.cli plan      --config run.json --objective roofline
  python -m paper_2311_00257_b200.cli import-profile profile.csv out.json

Exit codes: 0 ok, 1 configuration / profile error, 2 no
feasible plan (the report is still written). Reports are deterministic JSON
(sorted keys, shortest round-trip floats) that echo the resolved config.
Every computation goes through libamsp.so (the C++ planner).

RunConfig (unknown keys are rejected, with the offending path named):
  {"model":   {"llama": "llama-7b" | <ModelSpec fields>, "micro_batch": 1, ...},
   "cluster": {"gpus_per_node": 8, "node_count": 1, "gpu_memory_capacity": 8e10,
               "dp_mesh": [8, 1], "topology": {...}},
   "profile_path": "profiles/b200_nccl_4gpu.csv",      (optional; default: synthetic B200)
   "cost": {<CostConfig fields>}, "sim": {<SimConfig fields>}}
"""
from __future__ import annotations

import argparse
import json
import sys
from dataclasses import asdict, fields
from pathlib import Path

from . import _native as N
from . import shardplan as S

VERSION = "amsp-b200 r01"


class ConfigError(Exception):
    pass


def _check_keys(obj, allowed, path):
    if not isinstance(obj, dict):
        raise ConfigError(f"{path}: expected an object")
    for k in obj:
        if k not in allowed:
            raise ConfigError(f"{path}.{k}: unknown key")


def _mesh(v, path):
    if (not isinstance(v, (list, tuple)) or len(v) != 2 or
            not all(isinstance(x, int) and x >= 1 for x in v)):
        raise ConfigError(f"{path}: expected [per_node, nodes] of positive integers")
    return S.DeviceMesh(*v)


def parse_plan(text: str) -> S.ShardingPlan:
    parts = dict(kv.split("=") for kv in text.split(","))
    m = lambda s: S.DeviceMesh(*map(int, s.split("x")))  # noqa: E731
    return S.ShardingPlan(m(parts["p"]), m(parts["g"]), m(parts["os"]),
                          m(parts["p2"]) if "p2" in parts else None)


def load_config(path: str):
    try:
        raw = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise ConfigError(f"config: {e}") from e
    _check_keys(raw, {"model", "cluster", "profile_path", "cost", "sim"}, "config")
    model_f = {f.name for f in fields(S.ModelSpec)}
    mcfg = raw.get("model")
    if mcfg is None:
        raise ConfigError("config.model: missing")
    _check_keys(mcfg, model_f | {"llama"}, "config.model")
    if "llama" in mcfg:
        if mcfg["llama"] not in S.MODELS:
            raise ConfigError(f"config.model.llama: unknown model {mcfg['llama']!r}")
        kw = {k: mcfg[k] for k in ("micro_batch", "micro_batch_count", "seq_len") if k in mcfg}
        model = S.model(mcfg["llama"], **kw)
    else:
        model = S.ModelSpec(**mcfg)
    ccfg = raw.get("cluster")
    if ccfg is None:
        raise ConfigError("config.cluster: missing")
    _check_keys(ccfg, {"gpus_per_node", "node_count", "gpu_memory_capacity", "dp_mesh",
                       "topology"}, "config.cluster")
    topo = ccfg.get("topology", {})
    _check_keys(topo, {"leaf_count", "nodes_per_leaf", "inter_leaf_penalty"},
                "config.cluster.topology")
    R, Nn = ccfg.get("gpus_per_node", 8), ccfg.get("node_count", 1)
    cluster = S.ClusterSpec(R, Nn, int(ccfg.get("gpu_memory_capacity", 0)),
                            _mesh(ccfg.get("dp_mesh", [R, Nn]), "config.cluster.dp_mesh"),
                            S.Topology(topo.get("leaf_count", Nn), topo.get("nodes_per_leaf", 1),
                                       topo.get("inter_leaf_penalty", 1.0)))
    cost_f = {f.name for f in fields(S.CostConfig)}
    _check_keys(raw.get("cost", {}), cost_f, "config.cost")
    cost = S.CostConfig(**raw.get("cost", {}))
    sim_f = {f.name for f in fields(S.SimConfig)}
    _check_keys(raw.get("sim", {}), sim_f, "config.sim")
    sim = S.SimConfig(**raw.get("sim", {}))
    if sim.overlap_tier not in S.SimConfig.TIERS:
        raise ConfigError(f"config.sim.overlap_tier: unknown tier {sim.overlap_tier!r}")
    return raw, model, cluster, cost, sim


def load_profile(path):
    if path:
        return S.BandwidthProfile.load(path)
    from .engine import b200_profile
    return b200_profile()


def _result(r: S.PlanResult):
    return {"plan": str(r.plan), "time": asdict(r.time), "memory": asdict(r.memory),
            "feasible": r.feasible, "rank": r.rank}


def _emit(report, args):
    text = json.dumps(report, sort_keys=True, indent=2 if args.pretty else None)
    if args.out:
        Path(args.out).write_text(text + "\n")
    else:
        print(text)


def cmd_plan(args):
    raw, model, cluster, cost, sim = load_config(args.config)
    prof = load_profile(args.profile or raw.get("profile_path"))
    report = {"version": VERSION, "command": "plan", "config": raw}
    if args.objective == "roofline":
        return _plan_roofline(args, model, cluster, cost, prof, report)
    try:
        rep = S.solve(model, cluster, prof, cost, keep_all_results=args.all_candidates)
    except S.NoFeasiblePlanError as e:
        report.update(feasible=False, error=str(e), closest=_result(e.closest()))
        _emit(report, args)
        return 2
    report.update(feasible=True, best=_result(rep.best),
                  candidates_evaluated=rep.candidates_evaluated,
                  candidates_filtered=rep.candidates_filtered)
    if rep.all_results is not None:
        report["all_candidates"] = [_result(r) for r in rep.all_results]
    _emit(report, args)
    return 0


def _plan_roofline(args, model, cluster, cost, prof, report):
    """`plan --objective roofline`: the reference's candidates ranked by the
    engine's B200 step roofline (amsp_solve_roofline), not by T_comm."""
    report["objective"] = {"name": "roofline", "hbm_bytes_per_s": args.hbm_bw,
                           "nvlink_bytes_per_s": args.nvlink_bw}
    try:
        ranked = S.solve_roofline(model, cluster, prof, cost, args.hbm_bw, args.nvlink_bw)
    except S.NoFeasiblePlanError as e:
        report.update(feasible=False, error=str(e), closest=_result(e.closest()))
        _emit(report, args)
        return 2

    def row(r, st):
        return dict(_result(r), step_roofline=asdict(st))

    report.update(feasible=True, best=row(*ranked[0]), candidates_evaluated=len(ranked))
    if args.all_candidates:
        report["all_candidates"] = [row(r, st) for r, st in ranked]
    _emit(report, args)
    return 0


def cmd_roofline(args):
    """Per-rank algorithmic bytes and the B200 roofline step time of one
    engine step for a plan (default: the reference solver's pick), e.g. the
    8-GPU projections of DESIGN.md."""
    raw, model, cluster, cost, sim = load_config(args.config)
    if args.preset:
        plan = S.preset(args.preset, cluster)
    elif args.plan:
        plan = parse_plan(args.plan)
    else:
        plan = S.solve(model, cluster, load_profile(args.profile or raw.get("profile_path")),
                       cost).best.plan
    v = S.validate_plan(plan, cluster)
    if not v.ok():
        raise ConfigError("plan " + str(plan) + " violates " +
                          "; ".join(f"{x.constraint} ({x.detail})" for x in v.violations))
    tensors = S.model_tensors(model)
    dp = cluster.dp_mesh
    ranks = [asdict(S.step_roofline(tensors, plan, dp, r, gathers=args.gathers,
                                    hbm_bw=args.hbm_bw, nvlink_bw=args.nvlink_bw)[0])
             for r in range(dp.size())]
    worst, who = S.step_roofline(tensors, plan, dp, gathers=args.gathers, hbm_bw=args.hbm_bw,
                                 nvlink_bw=args.nvlink_bw)
    _emit({"version": VERSION, "command": "roofline", "config": raw, "plan": str(plan),
           "hbm_bytes_per_s": args.hbm_bw, "nvlink_bytes_per_s": args.nvlink_bw,
           "params": sum(tensors), "slowest_rank": who, "step": asdict(worst),
           "params_per_s_bound": sum(tensors) / worst.t_step, "ranks": ranks}, args)
    return 0


def cmd_simulate(args):
    raw, model, cluster, cost, sim = load_config(args.config)
    prof = load_profile(args.profile or raw.get("profile_path"))
    if args.overlap:
        sim.overlap_tier = args.overlap
    if args.preset:
        plan = S.preset(args.preset, cluster)
    elif args.plan:
        plan = parse_plan(args.plan)
    else:
        plan = S.solve(model, cluster, prof, cost).best.plan
    v = S.validate_plan(plan, cluster)
    if not v.ok():
        raise ConfigError("plan " + str(plan) + " violates " +
                          "; ".join(f"{x.constraint} ({x.detail})" for x in v.violations))
    res = S.simulate(model, cluster, plan, prof, cost, sim, with_trace=bool(args.trace))
    if args.trace:
        Path(args.trace).write_text(res.trace)
    peak = sim.peak_flops_per_gpu
    flops = 6.0 * model.total_params * model.micro_batch * model.seq_len * \
        model.micro_batch_count
    _emit({"version": VERSION, "command": "simulate", "config": raw, "plan": str(plan),
           "overlap_tier": sim.overlap_tier, "step_time": res.step_time,
           "compute_idle": res.compute_idle, "events": res.n_events,
           "mfu_param_flops": flops / (res.step_time * peak) if res.step_time > 0 else None,
           "comm": asdict(S.total_comm_time(model, cluster, plan, prof, cost)),
           "memory": asdict(S.memory_breakdown(model, plan, cost))}, args)
    return 0


def cmd_compare(args):
    raw, model, cluster, cost, sim = load_config(args.config)
    prof = load_profile(args.profile or raw.get("profile_path"))
    rows = []
    for name in S.preset_names():
        try:
            plan = S.preset(name, cluster)
        except S.InfeasibleError as e:
            rows.append({"name": name, "error": str(e)})
            continue
        row = {"name": name, "plan": str(plan),
               "time": asdict(S.total_comm_time(model, cluster, plan, prof, cost)),
               "memory": asdict(S.memory_breakdown(model, plan, cost))}
        row["feasible"] = row["memory"]["d_total"] <= cluster.gpu_memory_capacity
        row["simulated_step"] = S.simulate(model, cluster, plan, prof, cost, sim).step_time
        rows.append(row)
    try:
        best = S.solve(model, cluster, prof, cost).best
        rows.append({"name": "solver", "plan": str(best.plan), "time": asdict(best.time),
                     "memory": asdict(best.memory), "feasible": True,
                     "simulated_step": S.simulate(model, cluster, best.plan, prof, cost,
                                                  sim).step_time})
    except S.NoFeasiblePlanError as e:
        rows.append({"name": "solver", "error": str(e), "feasible": False})
    rows.sort(key=lambda r: (r.get("simulated_step") is None, r.get("simulated_step") or 0,
                             r["name"]))
    _emit({"version": VERSION, "command": "compare", "config": raw, "rows": rows}, args)
    return 0


def cmd_import_profile(args):
    prof = S.BandwidthProfile.from_csv(Path(args.csv).read_text())
    Path(args.out_json).write_text(prof.to_canonical_json())
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="amsp")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("plan", "simulate", "compare", "roofline"):
        p = sub.add_parser(name)
        p.add_argument("--config", required=True)
        p.add_argument("--profile", default=None)
        p.add_argument("--out", default=None)
        p.add_argument("--pretty", action="store_true")
        if name == "plan":
            p.add_argument("--all-candidates", action="store_true")
            p.add_argument("--objective", default="comm", choices=["comm", "roofline"],
                           help="comm: the reference solver (T_comm); roofline: the B200 "
                                "step roofline of the engine (HBM / NVLink bytes)")
            p.add_argument("--hbm-bw", type=float, default=S.B200_HBM_BW)
            p.add_argument("--nvlink-bw", type=float, default=S.B200_NVLINK_BW)
        if name in ("simulate", "roofline"):
            p.add_argument("--preset", default=None)
            p.add_argument("--plan", default=None)
        if name == "roofline":
            p.add_argument("--gathers", type=int, default=2)
            p.add_argument("--hbm-bw", type=float, default=S.B200_HBM_BW)
            p.add_argument("--nvlink-bw", type=float, default=S.B200_NVLINK_BW)
        if name == "simulate":
            p.add_argument("--overlap", default=None, choices=S.SimConfig.TIERS)
            p.add_argument("--trace", default=None)
    p = sub.add_parser("import-profile")
    p.add_argument("csv")
    p.add_argument("out_json")
    args = ap.parse_args(argv)
    try:
        return {"plan": cmd_plan, "simulate": cmd_simulate, "compare": cmd_compare,
                "roofline": cmd_roofline, "import-profile": cmd_import_profile}[args.cmd](args)
    except (ConfigError, N.InvalidConfig, S.InfeasibleError, KeyError, ValueError,
            TypeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
