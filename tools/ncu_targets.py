#!/usr/bin/env python
"""Small single-process drivers of the default AMSP kernels, for ncu
captures at HEAD (one GPU; W > 1 groups emulated in one process, so the
"peer" gradient reads and parameter stores hit local HBM -- the DRAM bytes
are the multi-GPU kernel's HBM + NVLink bytes landing on one device).

  python tools/ncu_targets.py fused  --world W [--model llama-1b] [--variant 0]
  python tools/ncu_targets.py gather --world W [--model llama-1b]   (ZeRO-3, TMA gather)
  python tools/ncu_targets.py push --world W [--model llama-1b]     (ZeRO-3 step: the
      push all-gather of unit 0, push_tma_kernel)
  python tools/ncu_targets.py staged --world W [--model llama-1b]   (ZeRO-2, M=2: the
      accumulate_kernel of micro-batch 0, then the fused update with accumulator sources)

Prints one JSON line: kernel name, variant, grid, per-launch algorithmic
bytes and CUDA-event ms per launch (outside ncu only).
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
    ap.add_argument("what", choices=["fused", "gather", "staged", "push"])
    ap.add_argument("--model", default="llama-1b")
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--unit", type=int, default=8, help="gather: the unit ncu captures")
    args = ap.parse_args()
    M = S.DeviceMesh
    W = args.world
    model = S.model(args.model)
    mb = 1
    if args.what == "fused":
        plan = S.ShardingPlan(M(1, 1), M(1, 1), M(W, 1))
    elif args.what == "staged":
        plan = S.ShardingPlan(M(1, 1), M(W, 1), M(W, 1))
        mb = 2
    else:
        plan = S.ShardingPlan(M(W, 1), M(W, 1), M(W, 1))
    engines = [Engine(model, plan, M(W, 1), rank=r, micro_batches=mb) for r in range(W)]
    if W > 1:
        link_local(engines)
    for e in engines:
        if args.variant:
            e.tune(args.variant)
        e.init_state()
        e.synth_grads(1)
    torch.cuda.synchronize()
    phi = engines[0].info.total_params
    info = engines[0]._info()
    out = {"what": args.what, "model": args.model, "phi": phi, "world": W,
           "variant": info.variant, "grid": info.grid}
    if args.what == "push":
        # one launch = this rank's slice of unit 0 read locally (2 B x unit / W)
        # and stored into the W members' slots (2 B x unit)
        ue = engines[0].unit(0)[2]
        out["algorithmic_bytes_per_launch"] = 2 * ue // W + 2 * ue
        for e in engines:
            e.time_kernel(True)
        for t in range(1, args.steps + 1):
            for e in engines:
                e.synth_grads(t)
            for e in engines:
                e.step(t)
        torch.cuda.synchronize()
        gms, gn = engines[0].gather_ms()
        out["gather_passes_ms"] = gms / max(gn, 1)
    elif args.what == "staged":
        # accumulate (rank 0): acc_elems x (2 B from each of the W G-block
        # ranks + 2 B accumulator write; first micro-batch: no read); fused:
        # owned x (2 B x W holders' accumulators... here W/s_g = 1 holder:
        # 2 B + 2 B x W raw grads + 24 B state + 2 B x W param stores)
        acc = info.acc_elems
        out["algorithmic_bytes_accumulate"] = acc * (2 * W + 2)
        out["algorithmic_bytes_per_launch"] = info.owned * (2 + 2 * W + 24 + 2 * W)
        for e in engines:
            e.time_kernel(True)
        for t in range(1, args.steps + 1):
            for k in range(mb):
                for e in engines:
                    e.synth_grads(t, mb=k)
                if k + 1 < mb:
                    for e in engines:
                        e.accumulate(t, k)
            for e in engines:
                e.step(t)
        torch.cuda.synchronize()
        ms, n = engines[0].kernel_ms()
        ams, an = engines[0].accum_ms()
        out["kernel_ms"] = ms / max(n, 1)
        out["accumulate_ms"] = ams / max(an, 1)
        out["variant"] = engines[0]._info().variant
    elif args.what == "fused":
        # per launch (rank 0): owned elements x (2 B grad from each of W ranks +
        # 24 B state r/w + 2 B param store into each of the W OS-group ranks)
        owned = info.owned
        out["algorithmic_bytes_per_launch"] = owned * (2 * W + 24 + 2 * W)
        for e in engines:
            e.time_kernel(True)
        for t in range(1, args.steps + 1):
            for e in engines:
                e.step(t)
        torch.cuda.synchronize()
        ms, n = engines[0].kernel_ms()
        out["kernel_ms"] = ms / max(n, 1)
        out["achieved_gbs"] = out["algorithmic_bytes_per_launch"] / (out["kernel_ms"] * 1e-3) / 1e9
    else:
        e = engines[0]
        # one all-gather pass of every unit: (s_p - 1)/s_p * 2 B pulled + 2 B
        # written per gathered element
        elems = sum(e.unit(u)[2] for u in range(info.n_units))
        out["units"] = info.n_units
        out["algorithmic_bytes_per_pass"] = int(elems * 2 * (W - 1) / W + 2 * elems)
        # the captured launch: unit `--unit` (ncu -s skips the earlier ones)
        ue = e.unit(args.unit)[2]
        out["algorithmic_bytes_per_unit"] = int(ue * 2 * (W - 1) / W + 2 * ue)
        for t in range(args.steps):
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            ev0.record(cur)
            for u in range(info.n_units):
                e.gather(u, u % 2, cur)
            ev1.record(cur)
            torch.cuda.synchronize()
            out["pass_ms"] = ev0.elapsed_time(ev1)
        out["achieved_gbs"] = out["algorithmic_bytes_per_pass"] / (out["pass_ms"] * 1e-3) / 1e9
    print(json.dumps(out), flush=True)
    for e in engines:
        e.close()


if __name__ == "__main__":
    main()
