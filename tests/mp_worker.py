"""torchrun worker for the multi-GPU parity test (one process per GPU).

  torchrun --nproc-per-node N tests/mp_worker.py --os-mesh Kx1 [--layout greedy]

Each rank runs the AMSP step over real NVLink peer memory (cudaIpc-mapped
buffers, device-side barriers) and checks its optimizer-state shard and its
full bf16 parameter copy bit-exactly against the CPU oracle."""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import cpu as O  # noqa: E402
from paper_2311_00257_b200 import shardplan as S  # noqa: E402
from paper_2311_00257_b200.engine import DEFAULT_SEED, Engine, pshard_layout  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--os-mesh", default=None)
    ap.add_argument("--dp-mesh", default=None)
    ap.add_argument("--layout", default="greedy")
    ap.add_argument("--p-mesh", default=None)
    ap.add_argument("--g-mesh", default=None,
                    help="explicit G mesh (default: the P mesh when given, else 1x1)")
    ap.add_argument("--micro-batches", type=int, default=1)
    ap.add_argument("--p2-mesh", default=None,
                    help="ZeRO++ secondary parameter mesh (backward all-gathers)")
    ap.add_argument("--synth", action="store_true",
                    help="scheduler: every grad-weight event writes its micro-batch gradient "
                         "during the step (grad_source=synth); no host barriers anywhere")
    ap.add_argument("--two-scheds", action="store_true",
                    help="run the steps through two schedulers created on the same engine, "
                         "alternating, with no host synchronisation between steps")
    ap.add_argument("--sched", action="store_true")
    ap.add_argument("--ring", action="store_true",
                    help="scheduler + s_g > 1: the gradient buffer is the schedule's smallest "
                         "ring (learned from a first engine with a generous ring)")
    ap.add_argument("--gather", default="sm", choices=["sm", "tma", "dma", "push"])
    ap.add_argument("--reduce", default="sm", choices=["sm", "dma"],
                    help="scheduler gradient reduce: SM NVLink pulls / copy-engine staged")
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--variant", type=int, default=0, help="fused-kernel variant (5/6 = TMA)")
    ap.add_argument("--full", action="store_true",
                    help="check every element at full model size, streamed in chunks "
                         "(tests/fullcheck.py) instead of materialising the whole model")
    ap.add_argument("--host", action="store_true",
                    help="amsp_engine_step_host: pinned host gradients, chunked H2D + per-chunk "
                         "barrier + fused update")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # More ranks than GPUs (W=8 on a 2- or 4-GPU box) places several ranks on
    # one device: the peer-memory path is the same (cudaIpc handles, flags),
    # only the timing is meaningless.
    local = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    M = S.DeviceMesh
    mesh = lambda s: M(*map(int, s.split("x")))  # noqa: E731
    dp = mesh(args.dp_mesh) if args.dp_mesh else M(world, 1)
    os_mesh = mesh(args.os_mesh) if args.os_mesh else dp
    p_mesh = mesh(args.p_mesh) if args.p_mesh else M(1, 1)
    g_mesh = p_mesh if p_mesh == os_mesh or args.p_mesh else M(1, 1)
    if args.g_mesh:
        g_mesh = mesh(args.g_mesh)
    MB = args.micro_batches
    plan = S.ShardingPlan(p_mesh, g_mesh, os_mesh,
                          secondary_params=mesh(args.p2_mesh) if args.p2_mesh else None)
    # "chunky": three raw tensors (300M params) so the host-buffer step spans
    # two 2^28-element upload chunks, with the chunk boundary inside a tensor.
    model = [200_000_000, 100_000_008, 64] if args.model == "chunky" else S.model(args.model)
    ring = 0
    if args.ring:
        from paper_2311_00257_b200.engine import Scheduler, b200_profile
        probe = Engine(model, plan, dp, rank=rank, device=local, layout=args.layout,
                       skip_gathers=True, micro_batches=MB,
                       grad_ring=S.model(args.model).total_params)
        probe.connect()
        ps = Scheduler(probe, S.model(args.model, micro_batch_count=MB), b200_profile(),
                       S.CostConfig(bucket_size=1 << 20),
                       S.SimConfig(overlap_tier="ag_rs_ar_bc", peak_flops_per_gpu=1e16),
                       grad_source="synth")
        ring = ps.info.grad_ring_need
        ps.close()
        probe.close()
        dist.barrier()
    e = Engine(model, plan, dp, rank=rank, device=local, layout=args.layout,
               skip_gathers=args.sched, micro_batches=MB, grad_ring=ring)
    e.connect()
    if args.variant:
        e.tune(args.variant)
    if plan.sp() > 1:
        e.tune_gather(args.gather)
    e.init_state()
    sched = None
    scheds = []
    if args.sched:  # overlap scheduler: real cross-GPU barriers per bucket / module
        from paper_2311_00257_b200.engine import Scheduler, b200_profile
        for _ in range(2 if args.two_scheds else 1):
            scheds.append(Scheduler(e, S.model(args.model, micro_batch_count=MB), b200_profile(),
                                    S.CostConfig(bucket_size=1 << 20),
                                    S.SimConfig(overlap_tier="ag_rs_ar_bc",
                                                peak_flops_per_gpu=1e16),
                                    gather=args.gather, reduce=args.reduce,
                                    grad_source="synth" if args.synth else "caller"))
        sched = scheds[0]
    for t in range(1, args.steps + 1):
        if sched and args.synth:
            # gradients appear inside the step (grad-weight events); the
            # device barriers alone order every cross-GPU read
            scheds[(t - 1) % len(scheds)].step(t)
        elif sched:
            e.synth_grads(t)
            dist.barrier()  # every rank's grads of step t exist before pulls
            sched.step(t)
            torch.cuda.synchronize()
            dist.barrier()
        elif MB > 1:
            e.micro_step(t)
        elif args.host:
            e.synth_grads(t)
            g = e.read("grads")  # this rank's step-t gradients, staged through host memory
            host = torch.from_numpy(g.view(np.int16)).pin_memory()
            e.step_host(t, host.data_ptr())
        else:
            e.synth_grads(t)
            e.step(t)
    if sched:
        scheds[(args.steps - 1) % len(scheds)].flush()  # mirrored broadcast: the last shards
        torch.cuda.synchronize()
        for s in scheds:
            s.close()
    torch.cuda.synchronize()
    if args.full:
        from fullcheck import check_engine
        per_proc = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        O.lib().amsp_o_set_threads(max(1, (os.cpu_count() or 1) // per_proc))
        bad = check_engine(e, args.steps, world, log=lambda m: print(f"RANK {rank} {m}",
                                                                     flush=True))
        for b in bad:
            print(f"RANK {rank} MISMATCH {b}", flush=True)
        e.close()
        dist.barrier()
        print(f"RANK {rank} {'OK' if not bad else 'FAIL'} full-size", flush=True)
        dist.destroy_process_group()
        sys.exit(0 if not bad else 1)
    phi = e.info.total_params
    segs, owned = e.segments()
    ok = True
    # a rank may own no tensor (greedy layout, fewer tensors than ranks)
    idx = np.concatenate([np.arange(f, f + ln, dtype=np.uint64) for f, _, ln in segs]
                         or [np.empty(0, np.uint64)])
    acc = O.accum(MB, plan.sg(), O.mesh_blocks((dp.per_node, dp.nodes),
                                                (g_mesh.per_node, g_mesh.nodes), world))
    want = (O.trajectory(idx, DEFAULT_SEED, args.steps, world, O.hyper(), acc) if owned
            else [[]] * 3)
    for name, ref in zip(("master", "exp_avg", "exp_avg_sq") if owned else (), want[:3]):
        got = e.read(name)
        if not np.array_equal(got.view(np.uint32), ref.view(np.uint32)):
            print(f"RANK {rank} MISMATCH {name}: {int(np.sum(got != ref))}", flush=True)
            ok = False
    params = e.read("params")
    full_all = O.trajectory_range(0, phi, DEFAULT_SEED, args.steps, world, O.hyper(), acc)[3]
    psegs, pn = pshard_layout(e.tensor_sizes, plan.sp(), e.info.p_position, 1, 0, "contiguous")
    full = np.empty(pn, np.uint16)
    for f, _, d, ln in psegs:
        full[d:d + ln] = full_all[f:f + ln]
    if plan.sp() > 1:  # every all-gather unit reproduces the updated tensors
        offs = np.cumsum([0] + e.tensor_sizes)
        for u in range(e.info.n_units):
            first, _, elems = e.unit(u)
            e.gather(u, 0)
            got = e.read("slot0", 0, elems)
            if not np.array_equal(got, full_all[offs[first]:offs[first] + elems]):
                print(f"RANK {rank} MISMATCH gather unit {u}", flush=True)
                ok = False
    if not np.array_equal(params, full):
        print(f"RANK {rank} MISMATCH params: {int(np.sum(params != full))}", flush=True)
        ok = False
    st = e.stats()
    e.close()
    dist.barrier()
    print(f"RANK {rank} {'OK' if ok else 'FAIL'} owned={owned} stats={st[0]:.4e}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
