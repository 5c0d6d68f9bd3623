"""All-gather pass microbenchmark over real NVLink (torchrun, one rank per GPU).

  torchrun --nproc-per-node 4 tools/tune_gather.py [--model llama-13b]

Times full forward all-gather passes (every unit) for several gather grids
and reports per-GPU ingress GB/s (2*Phi*(s_p-1)/s_p bytes per pass)."""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2311_00257_b200 import _native as N  # noqa: E402
from paper_2311_00257_b200 import shardplan as S  # noqa: E402
from paper_2311_00257_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-13b")
    ap.add_argument("--grids", default="0,-1,296,-1,0")
    ap.add_argument("--passes", type=int, default=4)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    M = S.DeviceMesh
    dp = M(world, 1)
    e = Engine(S.model(args.model), S.ShardingPlan(dp, dp, dp), dp, rank=rank, device=local,
               skip_gathers=True)
    e.connect()
    e.init_state()
    torch.cuda.synchronize()
    phi = e.info.total_params
    nbytes = 2 * phi * (world - 1) // world
    stream = torch.cuda.Stream()
    out = []
    for g in [int(x) for x in args.grids.split(",")]:
        N.check(N.lib().amsp_engine_tune_gather(e._h, g))
        for u in range(e.info.n_units):  # warm-up pass
            e.gather(u, u, stream)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.passes):
            for u in range(e.info.n_units):
                e.gather(u, u, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / args.passes
        dist.barrier()
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rec = {"grid": g, "pass_ms": round(float(t), 3),
               "ingress_GBps": round(nbytes / (float(t) * 1e-3) / 1e9, 1),
               "units": e.info.n_units, "wall_ms": round((time.perf_counter() - t0) * 1e3 / args.passes, 3)}
        out.append(rec)
        if rank == 0:
            print(json.dumps(rec), flush=True)
    e.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
