"""Sweep fused-kernel variants / grid sizes on one GPU (tuning aid).

  python tools/tune_fused.py [--model llama-7b] [--world 1] [--steps 5]

For world > 1 the DP group is emulated on one GPU (link_local), so NVLink is
not exercised; use bench.py under torchrun for that.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2311_00257_b200 import shardplan as S  # noqa: E402
from paper_2311_00257_b200.engine import Engine, link_local  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-7b")
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--variants", default="5,6")
    ap.add_argument("--grids", default="148,296")
    args = ap.parse_args()
    M = S.DeviceMesh
    model = S.model(args.model)
    W = args.world
    plan = S.ShardingPlan(M(1, 1), M(1, 1), M(W, 1))
    engines = [Engine(model, plan, M(W, 1), rank=r) for r in range(W)]
    if W > 1:
        link_local(engines)
    for e in engines:
        e.init_state()
        e.synth_grads(1)
    torch.cuda.synchronize()
    phi = engines[0].info.total_params
    out = []
    step = 0
    for v in [int(x) for x in args.variants.split(",")]:
        for g in [int(x) for x in args.grids.split(",")]:
            grid = engines[0].info.ntiles if g < 0 else g
            for e in engines:
                e.tune(v, grid)
            for e in engines:  # warm-up
                step += 1
                e.step(step)
            for e in engines:
                e.time_kernel(True)
            for _ in range(args.steps):
                step += 1
                for e in engines:
                    e.step(step)
            ms = sum(e.kernel_ms()[0] for e in engines) / args.steps
            for e in engines:
                e.time_kernel(False)
            bytes_ = sum(24 * e.info.owned for e in engines) + 4 * phi * W
            rec = {"variant": v, "chosen": engines[0].info.variant,
                   "grid": engines[0].info.grid, "ms": round(ms, 3),
                   "GBps": round(bytes_ / (ms * 1e-3) / 1e9, 1)}
            out.append(rec)
            print(json.dumps(rec), flush=True)
    best = min(out, key=lambda r: r["ms"])
    print(json.dumps({"best": best, "model": args.model, "world": W}))


if __name__ == "__main__":
    main()
