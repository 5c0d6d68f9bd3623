#!/usr/bin/env python
"""AMSP model-state step benchmark (BASELINE.json metric: "AMSP step ms &
params/s at 1/2/4/8 B200; collective bus GB/s vs NVLink").

A step = one pass of the AMSP model-state pipeline over LLaMA-7B model states
(bf16 P/G, fp32 master+m+v): cross-rank gradient reduce (fp32, fixed order)
with 1/W scale -> AdamW on this rank's OS shard -> bf16 params gathered into
every rank. Synthetic gradients (counter-based, oracle/amsp_oracle.c) are
resident in HBM when the timed region starts (`value`); `e2e` repeats the
step through the host-buffer C-ABI call (H2D of the step's gradients, D2H of
the step statistics inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

--impl reference times the reference's CPU implementation of the path. The
reference (`shardplan`) has no data plane, so that is the C/OpenMP
restatement in oracle/ ("port"), run on this box's host cores on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "AMSP step ms & params/s at 1/2/4/8 B200; collective bus GB/s vs NVLink"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
NVLINK_P2P_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "library"])
    ap.add_argument("--model", default="llama-7b")
    ap.add_argument("--plan", default="zero1",
                    help="zero1 (P/G replica, OS over dp) | replica | zero3 | roofline (the "
                         "native B200 roofline solver's pick) | 'p=AxB,g=AxB,os=AxB[,p2=AxB]' "
                         "(p2: ZeRO++ secondary parameter mesh)")
    ap.add_argument("--mesh", default=None, help="dp mesh per_node x nodes, default Nx1")
    ap.add_argument("--layout", default="greedy", choices=["greedy", "contiguous"])
    ap.add_argument("--variant", type=int, default=0, help="fused-kernel variant (0 auto)")
    ap.add_argument("--grid", type=int, default=0, help="fused-kernel grid (0 auto)")
    ap.add_argument("--overlap", action=argparse.BooleanOptionalAction, default=True,
                    help="also time the overlapped step (scheduler + compute stand-ins)")
    ap.add_argument("--tier", default="ag_rs_ar_bc", help="overlap tier for --overlap")
    ap.add_argument("--seq-len", type=int, default=4096)
    ap.add_argument("--micro-batch", type=int, default=1)
    ap.add_argument("--micro-batches", type=int, default=1,
                    help="M micro-batches per step: M-1 gradient accumulations into the G "
                         "shards (s_g > 1) before the fused update (PAPER.md:316-326)")
    ap.add_argument("--compute-eff", type=float, default=0.6)
    ap.add_argument("--comm-ctas", type=int, default=0)
    ap.add_argument("--trace-dir", default=None,
                    help="write measured + predicted TEF traces of one overlapped step here")
    ap.add_argument("--compute", default="both", choices=["standin", "gemm", "both"],
                    help="overlapped step compute: timed stand-ins or real cuBLAS GEMMs")
    ap.add_argument("--gemm-sm-margin", type=int, default=0,
                    help="SMs withheld from cuBLAS GEMMs for comm kernels (--compute gemm)")
    ap.add_argument("--optimizer-overlap", type=int, default=-1,
                    help="1: AdamW+push per bucket/module inside backward; 0: after the "
                         "barrier; -1: auto")
    ap.add_argument("--gather", default="dma", choices=["dma", "sm", "tma"],
                    help="overlapped all-gathers on copy engines (dma), the SM kernel or the "
                         "TMA bulk-copy kernel")
    ap.add_argument("--reduce", default="auto", choices=["auto", "sm", "dma"],
                    help="overlapped step's gradient reduces: SM NVLink pulls or copy-engine "
                         "staging (auto: dma when parameters are sharded, "
                         "profiles/r01_s2_overlap_reduce_dma_*.jsonl)")
    ap.add_argument("--bc", default="auto", choices=["auto", "push"],
                    help="overlapped step: mirrored broadcast of updated shards in the next "
                         "forward (auto, tier ag_rs_ar_bc) or push inside the optimizer")
    ap.add_argument("--step-gather", default="auto", choices=["auto", "sm", "dma", "tma", "push"],
                    help="all-gather implementation inside the pipeline-only step (s_p > 1); "
                         "auto = the engine's default (the TMA push kernel when the P slices are "
                         "aligned)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--grad-ring", action=argparse.BooleanOptionalAction, default=True,
                    help="s_g > 1: also time the overlapped step on a gradient-ring engine "
                         "(gradient memory = G shard + ring)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def mesh_of(s, S):
    a, b = s.lower().split("x")
    return S.DeviceMesh(int(a), int(b))


def plan_of(args, S, dp):
    if args.plan == "zero1":
        return S.ShardingPlan(S.DeviceMesh(1, 1), S.DeviceMesh(1, 1), dp)
    if args.plan == "replica":
        return S.ShardingPlan()
    if args.plan == "zero3":
        return S.ShardingPlan(dp, dp, dp)
    if args.plan == "roofline":
        # the native B200 roofline solver's pick (amsp_solve_roofline) for this
        # model on this mesh of 180 GB B200s
        from paper_2311_00257_b200.engine import b200_profile
        cl = S.ClusterSpec(dp.per_node, dp.nodes, 180_000_000_000, dp,
                           S.Topology(dp.nodes, 1, 1.0))
        return S.solve_roofline(S.model(args.model), cl, b200_profile())[0][0].plan
    parts = dict(kv.split("=") for kv in args.plan.split(","))
    return S.ShardingPlan(mesh_of(parts["p"], S), mesh_of(parts["g"], S), mesh_of(parts["os"], S),
                          secondary_params=mesh_of(parts["p2"], S) if "p2" in parts else None)


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def step_bytes(phi, owned, world, k, sp=1, sos=None, gathers=2, micro=1, acc_elems=0, sg=1,
               phases=False, s2=1):
    """Algorithmic bytes per GPU of ONE step (all ranks run concurrently;
    DESIGN.md §4). k = ranks sharing this rank's P position in its OS group
    (its parameter-store destinations), R = W/s_os replica groups.
    Fused reduce+AdamW+gather:
      HBM  = 24*owned (state r+w) + 2*Phi*R (owners' reads of this GPU's
             grads) + 2*Phi/s_p (parameter stores landing in this P shard)
      NVL in  = my pulls 2*owned*(W-1) + pushes into my P shard 2*(Phi/s_p-owned)
      NVL out = peers' pulls 2*(R*Phi-owned) + my pushes 2*owned*(k-1)
    s_p > 1 adds `gathers` all-gather passes (forward + backward):
      HBM  = 2*Phi (gathered write) + 2*Phi (the P group reading this shard)
      NVL  = 2*Phi*(s_p-1)/s_p per direction.
    M > 1 with s_g > 1 adds, per non-last micro-batch, the accumulation of
    the G shard (acc_elems bf16 accumulator elements on this rank, pulled
    from the s_g ranks of its G group):
      HBM  = 4*acc_elems (accumulator r/w) + 2*Phi (the holders read this
             GPU's gradients once)
      NVL in = 2*acc_elems*(s_g-1), out = 2*Phi*(s_g-1)/s_g
    and the last micro-batch's update reads the W/s_g holders' accumulators
    (2*owned each, W/s_g - 1 over NVLink) besides the raw gradients.
    ZeRO++ (s2 > 1): the backward pass gathers over the secondary group
    (2*Phi*(s2-1)/s2 per direction) and the forward pass refreshes the
    Phi/s2 secondary slice (4*Phi/s2 HBM).
    phases=True returns [(name, hbm, nvl)] per serial phase instead."""
    sos = sos or k * sp
    R = world // sos
    hbm = 24 * owned + 2 * phi * R + 2 * phi // sp
    nvl_in = 2 * owned * (world - 1) + 2 * (phi // sp - owned)
    nvl_out = 2 * (R * phi - owned) + 2 * owned * (k - 1)
    out = []
    if micro > 1 and sg > 1 and acc_elems:
        holders = world // sg
        a_hbm = (micro - 1) * (4 * acc_elems + 2 * phi) - 2 * acc_elems  # first: write only
        a_in = (micro - 1) * 2 * acc_elems * (sg - 1)
        a_out = (micro - 1) * 2 * phi * (sg - 1) // sg
        out.append(("accumulate", a_hbm, max(a_in, a_out) if world > 1 else 0))
        hbm += 2 * acc_elems
        nvl_in += 2 * owned * (holders - 1)
        nvl_out += 2 * acc_elems * (holders - 1)
    if world == 1:
        nvl_in = nvl_out = 0
    out.append(("update", hbm, max(nvl_in, nvl_out)))
    if sp > 1:
        gs = 1 if (s2 > 1 and gathers >= 2) else 0
        g_hbm = gathers * 4 * phi + (4 * phi // s2 if gs else 0)
        g_nvl = (gathers - gs) * 2 * phi * (sp - 1) // sp + (2 * phi * (s2 - 1) // s2 if gs else 0)
        out.insert(0, ("all_gather", g_hbm, g_nvl))
    if phases:
        return out
    return sum(x[1] for x in out), sum(x[2] for x in out)


def cpu_sample_size(phi_total):
    """The bounded CPU sample both arms use: 1/16 of the flat model (8-aligned),
    so one oracle step is ~0.1-0.3 s of host work."""
    return max(8, (phi_total // 16) // 8 * 8)


class CpuPort:
    """The oracle's CPU step (C + OpenMP, all host cores) on `n` consecutive
    params of the flat model: `world` ranks' bf16 gradients reduced in fixed
    order, 1/W scale, AdamW on one OS owner per element (ZeRO-1), the bf16
    params written into `world` copies (the gather). Test infrastructure:
    only bench.py's baseline legs run it."""

    def __init__(self, n, world):
        import numpy as np

        from oracle import cpu as O
        from paper_2311_00257_b200.engine import DEFAULT_SEED
        self.O, self.n, self.world = O, n, world
        self.cores = O.use_all_threads()
        self.h = O.hyper()
        self.grads = [O.grads(0, n, DEFAULT_SEED, 1, r) for r in range(world)]
        self.master = np.full(n, 0.01, np.float32)
        self.m = np.zeros(n, np.float32)
        self.v = np.zeros(n, np.float32)
        self.params = [np.zeros(n, np.uint16) for _ in range(world)]
        self.t = 0

    def step(self):
        self.t += 1
        self.O.step(self.grads, [(0, 0, self.n)], self.master, self.m, self.v, self.params,
                    self.O.scalars(self.t, self.world, self.h))

    def describe(self, phi_total, steps, secs):
        return (f"{self.n} consecutive params (1/16) of the {phi_total}-param flat model per "
                f"step: {self.world} rank gradients reduced + AdamW + bf16 into {self.world} "
                f"param copies; {steps} steps, {secs:.1f} s of CPU work")


def cpu_baseline(phi_total, world, steps_budget_s=10.0, max_steps=1000):
    """The oracle port timed on the bounded sample (cpu_sample_size) until
    about `steps_budget_s` of CPU work; value = sample params / median step."""
    port = CpuPort(cpu_sample_size(phi_total), world)
    port.step()  # warm-up (page-in)
    times = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < steps_budget_s and len(times) < max_steps:
        t0 = time.perf_counter()
        port.step()
        times.append(time.perf_counter() - t0)
    med = sorted(times)[len(times) // 2]
    return {"value": port.n / med, "unit": "params/s", "cores": port.cores, "kind": "port",
            "sample": port.describe(phi_total, len(times), sum(times)) +
                      f", median {med * 1e3:.1f} ms/step",
            "ms_per_step_full_workload_extrapolated": round(med * phi_total / port.n * 1e3, 1)}


def planner_timings(binary):
    """tests/cpp/plan_time.cpp (solve, build_schedule + simulate_step through
    the public shardplan API) run from `binary`: list of JSON records, or an
    error string."""
    if not Path(binary).exists():
        return f"{binary} not built"
    try:
        r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=120)
        if r.returncode != 0:
            return f"exit {r.returncode}: {r.stderr[-300:]}"
        return [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    except Exception as ex:  # reported, never required
        return str(ex)


def workload_config(args, S, world, phi):
    """The `config` object both arms print (same workload, same keys)."""
    dp = mesh_of(args.mesh, S) if args.mesh else S.DeviceMesh(world, 1)
    plan = plan_of(args, S, dp)
    mb = getattr(args, "micro_batches", 1)
    return {"workload": f"{args.model} model states ({phi} params: bf16 P/G, fp32 "
                        f"master+m+v), AMSP step = grad reduce + AdamW + param gather" +
                        (f", {mb} micro-batches (G-shard accumulation)" if mb > 1 else ""),
            "micro_batches": mb,
            "model": args.model, "phi": phi, "plan": str(plan), "dp_mesh": str(dp),
            "layout": args.layout,
            "l2": f"inputs ({(16 * phi) / 1e9:.0f} GB of model state) >> 126 MB L2",
            "parallelism": f"dp{world}"}


def run_reference(args):
    """The reference arm: the reference's CPU implementation of the path on
    this box's host cores. The reference (shardplan) is a planner/simulator
    with no data plane, so the step is the oracle's C/OpenMP restatement
    ("port") on a bounded sample; the reference's own compiled planner and
    simulator (oracle/_ref/plan_time_ref, built from /root/reference by
    oracle/build_ref.sh) are timed beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2311_00257_b200 import shardplan as S
    phi = S.model(args.model).total_params
    world = args.gpus
    port = CpuPort(cpu_sample_size(phi), world)
    for _ in range(args.warmup):
        port.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        port.step()
    dt = (time.perf_counter() - t0) / args.steps
    value = port.n / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32 (bf16 in/out)",
        "data": "synthetic",
        "config": workload_config(args, S, world, phi),
        "cpu_baseline": {"value": value, "unit": "params/s", "cores": port.cores, "kind": "port",
                         "sample": port.describe(phi, args.steps, dt * args.steps)},
        "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "ms_per_step_full_workload_extrapolated": round(dt * phi / port.n * 1e3, 1),
        "note": "a step = one oracle step over the bounded sample (value = sample params / "
                "step time); the reference (shardplan) is a CPU planner/simulator with no "
                "data plane, so its CPU path for this step is the oracle restatement "
                "(oracle/amsp_oracle.c)",
        "planner": planner_timings(REPO / "oracle" / "_ref" / "plan_time_ref"),
    }
    print(json.dumps(line), flush=True)


def run_library(args):
    """Library baseline of the same step (not the product): torch's fused
    AdamW (torch.optim.AdamW(fused=True)) on the fp32 master shard after an
    upcast, with NCCL reduce-scatter (fp32, the precision the oracle needs)
    and all-gather of bf16 params for W > 1 — what a ZeRO-1 framework on
    stock PyTorch + NCCL does. Prints one JSON line (impl library-baseline)."""
    import torch
    import torch.distributed as dist

    from paper_2311_00257_b200 import _native as N
    from paper_2311_00257_b200 import shardplan as S
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    phi = S.model(args.model).total_params
    shard = -(-phi // world)
    padded = shard * world
    grads = torch.empty(padded, dtype=torch.bfloat16, device=dev)
    N.check(N.lib().amsp_k_synth_grad(grads.data_ptr(), 0, phi, 0x414D5350, 1, rank, None))
    grads[phi:].zero_()
    params = torch.zeros(padded, dtype=torch.bfloat16, device=dev)
    master = torch.nn.Parameter(torch.full((shard,), 0.01, dtype=torch.float32, device=dev))
    opt = torch.optim.AdamW([master], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1,
                            fused=True)
    g32_full = torch.empty(padded, dtype=torch.float32, device=dev) if world > 1 else None
    stream = torch.cuda.current_stream()

    def step():
        if world > 1:
            g32_full.copy_(grads)                      # bf16 -> fp32 upcast
            g = torch.empty(shard, dtype=torch.float32, device=dev)
            dist.reduce_scatter_tensor(g, g32_full, op=dist.ReduceOp.SUM)
            g.mul_(1.0 / world)
            master.grad = g
        else:
            master.grad = grads[:shard].float()
        opt.step()
        mine = params[rank * shard:(rank + 1) * shard]
        mine.copy_(master.detach())                    # fp32 -> bf16 downcast
        if world > 1:
            dist.all_gather_into_tensor(params, mine.clone())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    if rank == 0:
        print(json.dumps({
            "impl": "library-baseline", "metric": METRIC, "value": phi / (ms * 1e-3),
            "unit": "params/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "config": {"workload": f"{args.model} model states, ZeRO-1 over {world}",
                       "path": "upcast + NCCL reduce_scatter(fp32) + torch fused AdamW + "
                               "downcast + NCCL all_gather(bf16)" if world > 1 else
                               "upcast + torch fused AdamW + downcast"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2311_00257_b200 import shardplan as S
    from paper_2311_00257_b200.engine import Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # More ranks than GPUs (e.g. --gpus 8 on a 4-GPU box) is a functional
    # check of the W-rank path only: ranks share devices, NCCL refuses
    # duplicate GPUs, so plumbing falls back to gloo and the line says so.
    oversub = world > torch.cuda.device_count()
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
    dp = mesh_of(args.mesh, S) if args.mesh else S.DeviceMesh(world, 1)
    model = S.model(args.model)
    plan = plan_of(args, S, dp)
    MB = args.micro_batches
    eng = Engine(model, plan, dp, rank=rank, device=local, layout=args.layout,
                 micro_batches=MB)
    eng.connect()
    if args.variant or args.grid:
        eng.tune(args.variant, args.grid)
    if args.step_gather != "auto":
        eng.tune_gather(args.step_gather)
    info = eng.info
    stream = torch.cuda.Stream(device=local)
    eng.init_state(stream)
    eng.synth_grads(1, stream)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if oversub else f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def amsp_step(t):
        # M-1 accumulations of the resident micro-batch gradients into the G
        # shards, then the fused update (the backward that would rewrite the
        # gradient buffer between micro-batches is not part of the pipeline)
        for k in range(MB - 1):
            eng.accumulate(t, k, stream)
        eng.step(t, stream)

    step = 0
    for _ in range(args.warmup):
        step += 1
        amsp_step(step)
    torch.cuda.synchronize()
    barrier()

    # Timed region: K device-resident steps; per-step CUDA events on the
    # engine stream for the step, and kernel-only events from the engine.
    launches0 = eng.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    eng.time_kernel(True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step += 1
            amsp_step(step)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = eng.launch_count() - launches0
    total_ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_per_step = total_ms / args.steps

    # The fused kernel alone (barriers excluded), bracketed by CUDA events on
    # the engine stream inside the same timed region.
    # Raises if a cross-GPU barrier of the timed steps timed out (device
    # error flag); a run with a lost peer never reports a number.
    eng.stats()
    k_total, k_n = eng.kernel_ms()
    g_total, g_n = eng.gather_ms()
    a_total, a_n = eng.accum_ms()
    eng.time_kernel(False)
    kernel_ms = max_over_ranks(k_total / max(k_n, 1))
    gather_ms = max_over_ranks(g_total / g_n) if g_n else 0.0
    accum_ms = max_over_ranks(a_total / args.steps) if a_n else 0.0  # per step

    phi = info.total_params
    value = phi / (ms_per_step * 1e-3)
    pk, pk_src = peaks()
    sb = dict(sp=info.sp, sos=plan.sos(), micro=MB, acc_elems=info.acc_elems, sg=plan.sg(),
              s2=info.secondary_shards)
    hbm_b, nvl_b = step_bytes(phi, info.owned, world, info.os_group_size, **sb)
    phases = step_bytes(phi, info.owned, world, info.os_group_size, phases=True, **sb)
    # s_p = 1, M = 1: the step is one fused launch (+2 tiny barriers) -> time
    # the kernel. s_p > 1 or M > 1: the all-gather passes / accumulations are
    # part of the roofline bytes, so the whole step is the timed unit.
    whole = info.sp > 1 or (MB > 1 and info.acc_elems > 0)
    t_meas = ms_per_step if whole else kernel_ms
    kname = "fused_step_tma_kernel" if info.variant >= 5 else "fused_step_kernel"
    scope = (f"{kname} (reduce + AdamW + gather), variant {info.variant}" if not whole else
             "whole step: " +
             ("2 all-gather passes (" +
              {"sm": "gather_kernel", "dma": "copy engines", "tma": "gather_tma_kernel",
               "push": "push_tma_kernel (NVLink stores)",
               "auto": "engine default: push_tma_kernel when aligned"}[args.step_gather] +
              ") + " if info.sp > 1 else "") +
             (f"{MB - 1} G-shard accumulations (accumulate_kernel) + " if MB > 1 else "") +
             "fused reduce/AdamW + barriers")
    hbm_ach = hbm_b / (t_meas * 1e-3) / 1e9
    nvl_ach = nvl_b / (t_meas * 1e-3) / 1e9
    t_hbm = hbm_b / (pk["hbm_gbs"] * 1e9)
    t_nvl = nvl_b / (NVLINK_P2P_GBS * 1e9)
    bound = "hbm" if t_hbm >= t_nvl else "nvlink"
    roof = {
        "bound": bound,
        "achieved": round(hbm_ach if bound == "hbm" else nvl_ach, 1),
        "peak": pk["hbm_gbs"] if bound == "hbm" else NVLINK_P2P_GBS,
        "unit": "GB/s",
        "frac": round((hbm_ach / pk["hbm_gbs"]) if bound == "hbm" else (nvl_ach / NVLINK_P2P_GBS), 4),
        "traffic": None,
        "kernel": scope,
        "kernel_ms": round(kernel_ms, 4),
        "timed_ms": round(t_meas, 4),
        "step_breakdown_ms": {"all_gather_passes": round(gather_ms, 4),
                              "g_shard_accumulations": round(accum_ms, 4),
                              "fused_reduce_adamw_gather": round(kernel_ms, 4),
                              "barriers_and_gaps": round(ms_per_step - gather_ms - accum_ms -
                                                         kernel_ms, 4)},
        "algorithmic_bytes": {"hbm": hbm_b, "nvlink_per_direction": nvl_b},
        "hbm": {"achieved": round(hbm_ach, 1), "peak": pk["hbm_gbs"],
                "frac": round(hbm_ach / pk["hbm_gbs"], 4), "peak_source": pk_src},
        "nvlink": {"achieved": round(nvl_ach, 1), "peak": NVLINK_P2P_GBS,
                   "frac": round(nvl_ach / NVLINK_P2P_GBS, 4),
                   "peak_source": "measured peer copy 770 GB/s/direction (B200_PROFILING.md); "
                                  "900 nominal"},
        "lower_bound_ms": round(max(t_hbm, t_nvl) * 1e3, 3),
        "frac_of_roofline_step": round(max(t_hbm, t_nvl) * 1e3 / ms_per_step, 4),
    }
    if len(phases) > 1:
        # The phases (all-gathers, accumulations, update) run one after the
        # other in the pipeline-only step: each is bound by its own
        # max(HBM, NVLink) time, and the step by their sum.
        pb = [{"phase": n, "hbm_bytes": h, "nvlink_bytes_per_direction": v,
               "bound_ms": round(max(h / (pk["hbm_gbs"] * 1e9), v / (NVLINK_P2P_GBS * 1e9)) *
                                 1e3, 3)} for n, h, v in phases]
        roof["phase_bounds"] = pb
        roof["phase_bound_ms"] = round(sum(x["bound_ms"] for x in pb), 3)
        roof["frac_of_phase_bound"] = round(roof["phase_bound_ms"] / ms_per_step, 4)
        roof["bound_note"] = ("lower_bound_ms assumes the phases overlap (sum of bytes / peak); "
                              "phase_bound_ms is the serial pipeline's bound")
    ncu_traffic = REPO / "profiles" / "r02_traffic.json"
    if ncu_traffic.exists() and not whole:
        try:
            d = json.loads(ncu_traffic.read_text())
            key = f"{args.model}/{world}"
            if key in d:
                roof["traffic"] = d[key]
            elif str(world) in d.get("ratio_by_world", {}):
                # ncu profiles one GPU per command, so a multi-rank step has no
                # capture: report the DRAM-traffic / algorithmic-bytes ratio of
                # the same default kernel with the W-rank group emulated on one
                # GPU (re-reads would show there), not an absolute figure
                rw = d["ratio_by_world"][str(world)]
                roof["traffic_over_algorithmic_emulated"] = rw["traffic_over_algorithmic"]
                roof["traffic_note"] = (f"{rw['kernel']}: ncu DRAM bytes / algorithmic bytes of "
                                        f"one launch with W={world} emulated on one GPU "
                                        f"({rw['source']})")
        except Exception:
            pass

    # Busbw of the collective the fused kernel implements (nccl-tests
    # convention: RS/AG (n-1)/n on the gathered size; AR 2(n-1)/n).
    # The fused kernel performs the reduce-scatter and the all-gather
    # concurrently in one launch, i.e. an all-reduce of the 2*Phi-byte bf16
    # gradient buffer (values in, updated values out): ONE busbw, AR
    # convention 2(n-1)/n * bytes / time.
    busbw = None
    if world > 1 and info.sp == 1:
        bw = 2 * (world - 1) / world * 2 * phi / (kernel_ms * 1e-3) / 1e9
        busbw = {"allreduce_equiv_busbw_gbs": round(bw, 1),
                 "convention": "nccl-tests AR: 2(n-1)/n x 2*Phi bytes / fused-kernel time "
                               "(RS + AG in one launch)",
                 "vs_nvlink_p2p_gbs": NVLINK_P2P_GBS, "vs_nvlink_nominal_gbs": NVLINK_NOMINAL_GBS,
                 "frac_of_nominal": round(bw / NVLINK_NOMINAL_GBS, 4)}
    # This box's NVLink peer-read peak, measured in-run after the timed
    # region (every rank pulls an equal share from every peer; the slowest
    # rank's ingress).
    nvl_probe = None
    if world > 1 and not oversub:
        try:
            ingress = eng.nvlink_probe(1 << 32, "all")
            nvl_probe = -max_over_ranks(-ingress)
            roof["nvlink"]["peak_measured_in_run_gbs"] = round(nvl_probe, 1)
            roof["nvlink"]["frac_of_measured_peak"] = round(nvl_ach / nvl_probe, 4)
            if busbw:
                busbw["nvlink_peer_read_measured_gbs"] = round(nvl_probe, 1)
        except Exception as ex:  # reported, never required
            roof["nvlink"]["peak_measured_in_run_error"] = str(ex)

    # Overlapped step: the reference event graph replayed by the scheduler on
    # 3 streams; measured with real cuBLAS GEMM compute (the realistic case)
    # and with the reference's timed stand-ins (6*Phi*B*S FLOPs at the
    # measured sustained bf16 peak x efficiency).
    def measure_overlap(compute, eng=eng, ring=False):
        nonlocal step
        from paper_2311_00257_b200.engine import Scheduler, b200_profile
        mspec = S.model(args.model, micro_batch=args.micro_batch, seq_len=args.seq_len,
                        micro_batch_count=MB)
        peak_tf = pk.get("bf16_tflops_sustained", 1400.0)
        sim = S.SimConfig(overlap_tier=args.tier, peak_flops_per_gpu=peak_tf * 1e12,
                          compute_efficiency=args.compute_eff)
        # Defaults from the r01 sweeps (profiles/r01_tune_overlap_*.jsonl):
        # with real GEMMs the HBM-bound optimizer competes with compute for
        # SMs, so it stays after the barrier unless P is sharded; all-gathers
        # run on the copy engines (no SMs taken from compute).
        opt = args.optimizer_overlap
        if opt < 0:
            opt = 1 if (compute == "standin" or plan.sp() > 1) else 0
        # Copy-engine staged reduces free the SMs for the GEMMs when P is
        # sharded (13B ZeRO-3 W=4: 283 vs 295 ms); with s_p = 1 the bucket
        # reduces share the copy engines with the mirrored broadcast and the
        # SM pulls win (7B ZeRO-1 W=4: 139.5 vs 150.6 ms).
        reduce = args.reduce if args.reduce != "auto" else ("dma" if plan.sp() > 1 else "sm")
        ctas = args.comm_ctas or (64 if (compute == "gemm" and plan.sp() > 1 and reduce == "sm")
                                  else 128)
        sched = Scheduler(eng, mspec, b200_profile(), S.CostConfig(), sim, comm_ctas=ctas,
                          optimizer_overlap=bool(opt), compute=compute,
                          gemm_sm_margin=args.gemm_sm_margin, gather=args.gather, bc=args.bc,
                          reduce=reduce,
                          grad_source=("synth" if ((MB > 1 or ring) and compute == "standin")
                                       else "caller"))

        def timed(with_comm, k):
            nonlocal step
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(k):
                step += 1
                sched.step(step, stream, with_comm)
            b.record(stream)
            torch.cuda.synchronize()
            barrier()
            return max_over_ranks(a.elapsed_time(b) / k)

        # FLOPs of the compute stream per step: the reference's compute model
        # (overlap_sim.cpp:97-110, flops_coeff_param 6 / flops_coeff_attn 12)
        # and, for compute='gemm', what the kernels execute (linear modules
        # incl. the LM head at 6 FLOPs/param/token, no embedding GEMM; the
        # attention GEMMs compute the full S x S square = 12*B*S^2*H/layer).
        toks = args.micro_batch * args.seq_len * MB
        H, L, S_ = mspec.hidden, mspec.layer_count, args.seq_len
        attn = 12.0 * L * args.micro_batch * MB * S_ * S_ * H
        lin_params = phi - mspec.vocab * H - (2 * L + 1) * H  # minus embedding and norms
        flops = {"model_6PhiBS_plus_attention": 6.0 * phi * toks + attn,
                 "total": (6.0 * lin_params * toks + attn) if compute == "gemm"
                 else 6.0 * phi * toks + attn}
        flops["executed_over_model"] = round(
            flops["total"] / flops["model_6PhiBS_plus_attention"], 4)
        timed(True, args.warmup)
        t_b = timed(True, args.steps)
        t_c = timed(False, args.steps)
        t_o = timed("optimizer", args.steps)
        si = sched.info
        if args.trace_dir:
            # One extra traced step (outside the timed regions): measured and
            # predicted Chrome traces with the reference's schema.
            sched.enable_trace(True)
            step += 1
            sched.step(step, stream, True)
            if rank == 0:
                text, _ = sched.trace()
                Path(args.trace_dir).mkdir(parents=True, exist_ok=True)
                tag = (f"{args.model}_w{world}_{str(plan).replace(',', '_').replace('=', '')}"
                       f"_{compute}")
                (Path(args.trace_dir) / f"measured_{tag}.json").write_text(text)
                (Path(args.trace_dir) / f"predicted_{tag}.json").write_text(
                    sched.predicted_trace())
        try:
            eng.stats()  # barrier error flag of the scheduled steps
        except Exception as ex:
            import re
            m = re.search(r"barrier id (\d+)", str(ex))
            if m and int(m.group(1)) >= 16:
                ev, role, mbi = sched.barrier_owner(int(m.group(1)))
                raise RuntimeError(f"{ex} -> scheduler event {ev} of {si.n_events}, {role} "
                                   f"barrier, micro-batch {mbi}, compute={compute}") from ex
            raise
        sched.close()
        return {"compute": compute, "tier": args.tier,
                "tokens_per_microbatch": args.micro_batch * args.seq_len,
                "optimizer": "in backward (per bucket/module)" if opt
                             else "after the step barrier (paper)",
                "gather": {"dma": "copy engines", "sm": "SM kernel",
                           "tma": "TMA bulk-copy kernel"}[args.gather],
                "comm_ctas": ctas,
                "reduce": {"sm": "SM kernels pull peers' gradients over NVLink",
                           "dma": "copy engines stage peers' gradients, SM kernels reduce "
                                  "locally"}[reduce],
                "param_broadcast": ("mirrored: copy-engine pulls in the next step's BC events, "
                                    "gating forward layer blocks" if si.mirrored_bc else
                                    "pushed by the optimizer kernels (NVLink stores)"),
                "step_ms": round(t_b, 3), "compute_only_ms": round(t_c, 3),
                "compute_plus_optimizer_ms": round(t_o, 3),
                # a step faster than its own no-communication baseline is
                # run-to-run noise (W = 1 has no communication at all): the
                # reported exposure is floored at 0, the raw difference kept
                "exposed_comm_ms": round(max(0.0, t_b - t_o), 3),
                "exposed_comm_frac": round(max(0.0, t_b - t_o) / t_b, 4),
                "exposed_comm_raw_ms": round(t_b - t_o, 3),
                "exposed_frac": round(max(0.0, t_b - t_c) / t_b, 4),
                "predicted_step_ms": round(si.predicted_step_s * 1e3, 3),
                "predicted_compute_ms": round(si.predicted_compute_s * 1e3, 3),
                "events": si.n_events, "buckets": si.n_buckets, "gathers": si.n_gather,
                "reduces": si.n_reduce, "barriers": si.n_barriers,
                "compute_model": (f"timed stand-ins: (6*Phi*B*S + 12*L*B*S^2*H) FLOPs at "
                                  f"{peak_tf} TF/s x {args.compute_eff}" if compute == "standin"
                                  else "real layer compute: cuBLAS bf16 GEMMs of every linear "
                                  "module (fwd, dgrad, wgrad into the gradient buffer), the "
                                  "attention core (strided-batched QK^T / PV GEMMs + causal "
                                  "softmax, and their backward) in the o-projection's events, "
                                  "RMSNorm kernels (fwd, dgrad, weight grad into the gradient "
                                  "buffer) for the norm modules"),
                "compute_flops": flops,
                "compute_only_tflops": round(flops["total"] / (t_c * 1e-3) / 1e12, 1),
                "profile": "synthetic B200 NVLink alpha-beta (680 GB/s, 5 us)"}

    overlap = None
    if args.overlap:
        modes = ["gemm", "standin"] if args.compute == "both" else [args.compute]
        results = [measure_overlap(c) for c in modes]
        overlap = results[0]
        if len(results) > 1:
            overlap = dict(results[0], standin=results[1])
        overlap["exposed_definitions"] = (
            "exposed_comm = step - (compute + local optimizer, no NVLink); exposed_frac = "
            "(step - compute only) / step, i.e. communication AND optimizer time not hidden")

    # End-to-end through the host-buffer C-ABI call.
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        host = torch.empty(phi, dtype=torch.int16, pin_memory=True)
        grads_dev = torch.empty(phi, dtype=torch.int16, device=f"cuda:{local}")
        # stage this rank's synthetic gradients into pinned host memory (setup)
        from paper_2311_00257_b200 import _native as N
        N.check(N.lib().amsp_k_synth_grad(grads_dev.data_ptr(), 0, phi, eng.seed, 1, rank,
                                          None))
        host.copy_(grads_dev)
        del grads_dev
        torch.cuda.synchronize()
        barrier()
        if MB > 1:
            # M micro-batches: each one's host gradients are copied (pinned,
            # async, on the engine stream) into the engine's gradient buffer,
            # then accumulated (k < M-1) or stepped (the last); D2H = stats
            class _Dev:  # the engine's gradient buffer as a torch tensor (no copy)
                __cuda_array_interface__ = {"shape": (phi,), "typestr": "<i2",
                                            "data": (info.grads, False), "version": 3}
            grads_view = torch.as_tensor(_Dev(), device=f"cuda:{local}")

            def host_step(t):
                with torch.cuda.stream(stream):
                    for k in range(MB):
                        grads_view.copy_(host, non_blocking=True)
                        if k + 1 < MB:
                            eng.accumulate(t, k, stream)
                    eng.step(t, stream)
                eng.stats()
        else:
            def host_step(t):
                eng.step_host(t, host.data_ptr(), stream)
        host_step(step + 1)
        step += 1
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            step += 1
            host_step(step)
        barrier()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": phi / e2e_s, "unit": "params/s", "ms_per_step": round(e2e_s * 1e3, 3),
               "h2d_bytes_per_step": 2 * phi * world * MB, "d2h_bytes_per_step": 8 * world,
               "steps": args.e2e_steps,
               "path": (f"{MB} micro-batches: pinned host bf16 grads -> async H2D into the "
                        "engine's gradient buffer -> amsp_engine_accumulate (k < M-1) / "
                        "amsp_engine_step (last) -> D2H stats" if MB > 1 else
                        "amsp_engine_step_host: pinned host bf16 grads -> chunked H2D (2^28 "
                        "elements) on a copy stream, each chunk's fused update (W > 1: after a "
                        "cross-GPU barrier) behind it -> D2H stats"
                        if info.sp == 1 else
                        "amsp_engine_step_host: pinned host bf16 grads -> H2D -> step -> "
                        "D2H stats"),
               "direction": "host gradients in, updated parameters stay on the device (the "
                            "D2H bytes are the step statistics)"}
        del host

    # Memory: this rank's device allocation against the planner's model-state
    # bytes (memory_breakdown, cost_model.cpp:140-160).
    mbd = S.memory_breakdown(S.model(args.model, micro_batch_count=MB), plan)
    memory = {"device_bytes": info.device_bytes, "grad_buffer_elems": info.grad_elems,
              "g_shard_accumulator_elems": info.acc_elems,
              "planner_d_modelstate": mbd.d_modelstate, "planner_d_grads": mbd.d_grads}

    # Gradient ring (s_g > 1): the overlapped step once more on an engine
    # whose gradient buffer is only the schedule's ring, so per-GPU gradient
    # memory is the G shard (D_g = 2*Phi/s_g) plus that transient ring.
    overlap_ring = None
    if args.overlap and plan.sg() > 1 and args.grad_ring:
        eng.close()
        from paper_2311_00257_b200.engine import Scheduler, b200_profile
        ring, need = max(info.owned, 1 << 26), None
        for _ in range(3):
            # probe: a scheduler on a ring too small reports the size it needs;
            # the measured engine gets exactly the schedule's smallest ring
            eng = Engine(model, plan, dp, rank=rank, device=local, layout=args.layout,
                         micro_batches=MB, skip_gathers=True, grad_ring=ring)
            eng.connect()
            if need is not None:
                break
            try:
                probe = Scheduler(eng, S.model(args.model, micro_batch=args.micro_batch,
                                               seq_len=args.seq_len, micro_batch_count=MB),
                                  b200_profile(), S.CostConfig(),
                                  S.SimConfig(overlap_tier=args.tier), grad_source="synth")
                need = probe.info.grad_ring_need
                probe.close()
            except Exception as ex:
                import re
                m = re.search(r"it needs (\d+)", str(ex))
                if not m:
                    raise
                need = int(m.group(1))
            ring = need
            eng.close()
        eng.init_state(stream)
        torch.cuda.synchronize()
        rinfo = eng._info()
        modes = ["gemm", "standin"] if args.compute == "both" else [args.compute]
        res = [measure_overlap(c, eng, ring=True) for c in modes]
        overlap_ring = dict(res[0], standin=res[1]) if len(res) > 1 else res[0]
        overlap_ring["memory"] = {"device_bytes": rinfo.device_bytes,
                                  "grad_ring_elems": rinfo.grad_elems, "ring_need_elems": need,
                                  "g_shard_accumulator_elems": rinfo.acc_elems,
                                  "saved_vs_full_gradient_bytes":
                                      info.device_bytes - rinfo.device_bytes}

    cpu = None
    planner = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(phi, world, steps_budget_s=10.0)
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"error": str(ex)}
        from paper_2311_00257_b200 import build as B
        planner = {"ours": planner_timings(B.PLAN_TIME),
                   "reference": planner_timings(REPO / "oracle" / "_ref" / "plan_time_ref")}

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "params/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32 (bf16 grads/params)", "data": "synthetic",
            "config": workload_config(args, S, world, phi),
            "roofline": roof, "busbw": busbw, "overlap": overlap,
            "overlap_grad_ring": overlap_ring, "memory": memory, "e2e": e2e,
            "cpu_baseline": cpu, "planner": planner,
            "gpu_launches": launches, "clocks": clk,
        }
        if oversub:
            line["oversubscribed"] = (f"{world} ranks on {torch.cuda.device_count()} GPUs: "
                                      "functional check, not a measurement")
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "library":
        run_library(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
