"""Sweep overlap knobs of the scheduler (comm CTAs, GEMM SM margin,
optimizer placement) on one engine (torchrun, one rank per GPU).

  torchrun --nproc-per-node 4 tools/tune_overlap.py --plan zero1 --compute gemm
"""
import argparse
import itertools
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2311_00257_b200 import shardplan as S  # noqa: E402
from paper_2311_00257_b200.engine import Engine, Scheduler, b200_profile  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-7b")
    ap.add_argument("--plan", default="zero1")
    ap.add_argument("--compute", default="gemm")
    ap.add_argument("--comm-ctas", default="32,64,128")
    ap.add_argument("--margins", default="0,16,32")
    ap.add_argument("--opt", default="1")
    ap.add_argument("--gather", default="sm")
    ap.add_argument("--opt-variant", default="0", help="in-backward optimizer kernel(s): 0 LDG, 5/6 TMA")
    ap.add_argument("--reduce", default="sm", help="gradient reduce: sm (NVLink pulls) / dma (staged)")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--seq-len", type=int, default=4096)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    M = S.DeviceMesh
    dp = M(world, 1)
    plan = {"zero1": S.ShardingPlan(M(1, 1), M(1, 1), dp), "zero3": S.ShardingPlan(dp, dp, dp),
            "zero2": S.ShardingPlan(M(1, 1), dp, dp),
            "replica": S.ShardingPlan()}[args.plan]
    model = S.model(args.model, seq_len=args.seq_len)
    eng = Engine(model, plan, dp, rank=rank, device=local)
    eng.connect()
    stream = torch.cuda.Stream()
    eng.init_state(stream)
    eng.synth_grads(1, stream)
    step = 0

    def timed(sched, with_comm, k):
        nonlocal step
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            step += 1
            sched.step(step, stream, with_comm)
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / k])
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    sim = S.SimConfig(peak_flops_per_gpu=1413.6e12, compute_efficiency=0.6)
    margins = args.margins.split(",")
    for cc, mg, oo, ga, ov, rd in itertools.product(
            [int(x) for x in args.comm_ctas.split(",")], margins,
            [int(x) for x in args.opt.split(",")], args.gather.split(","),
            [int(x) for x in args.opt_variant.split(",")], args.reduce.split(",")):
        mg = cc if mg == "cc" else int(mg)  # "cc": withhold exactly the comm CTAs' SMs
        sched = Scheduler(eng, model, b200_profile(), S.CostConfig(), sim, comm_ctas=cc,
                          optimizer_overlap=bool(oo), compute=args.compute, gemm_sm_margin=mg,
                          gather=ga, optimizer_variant=ov, reduce=rd)
        timed(sched, True, 1)
        tb = timed(sched, True, args.steps)
        tc = timed(sched, False, args.steps)
        to = timed(sched, "optimizer", args.steps)
        if rank == 0:
            print(json.dumps({"comm_ctas": cc, "gemm_sm_margin": mg, "optimizer_overlap": oo,
                              "gather": ga, "optimizer_variant": ov, "reduce": rd,
                              "step_ms": round(tb, 2), "compute_only_ms": round(tc, 2),
                              "compute_plus_optimizer_ms": round(to, 2),
                              "exposed_comm_frac": round((tb - to) / tb, 4),
                              "exposed_frac": round((tb - tc) / tb, 4)}), flush=True)
        sched.close()
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
