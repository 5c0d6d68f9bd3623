#!/usr/bin/env python
"""Bandwidth of the raw C-ABI kernels (include/amsp_c.h "kernels" section)
on one GPU: amsp_k_adamw (bf16 and fp32 grads), amsp_k_upcast_scale,
amsp_k_rs_upcast_scale (W local sources) and amsp_k_ag_downcast (k local
destinations), each timed with CUDA events on the launching stream over
`--iters` launches after warm-up. Sizes are far above the 126 MB L2.

Algorithmic bytes per element:
  adamw bf16 grad: 2 + 24 + 2 (param out) = 28   fp32 grad: 4 + 24 + 2 = 30
  upcast_scale:    2 + 4 = 6
  rs_upcast_scale: 2*W + 4
  ag_downcast:     4 + 2*k

  python tools/bench_raw.py [--n 268435456] [--iters 20] > raw.jsonl
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2311_00257_b200 import _native as N
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    n = args.n
    L = N.lib()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    sp = C.c_void_p(stream.cuda_stream)
    peaks = {}
    pf = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if pf.exists():
        peaks = json.loads(pf.read_text())
    hbm = peaks.get("hbm_gbs", 6650.0)

    g16 = torch.randn(n, device=dev).to(torch.bfloat16)
    g32 = torch.randn(n, device=dev)
    master = torch.randn(n, device=dev) * 0.02
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    p16 = torch.empty(n, dtype=torch.bfloat16, device=dev)
    out32 = torch.empty(n, device=dev)

    def timeit(name, fn, nbytes):
        if args.only and args.only not in name:
            return
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                fn()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.iters):
                fn()
            b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": name, "n": n, "ms": round(ms, 4),
                          "algorithmic_bytes": nbytes, "achieved_gbs": round(gbs, 1),
                          "hbm_peak_gbs": hbm, "frac": round(gbs / hbm, 4)}), flush=True)

    t = [0]

    def adamw(bf16):
        def f():
            t[0] += 1
            N.check(L.amsp_k_adamw((g16 if bf16 else g32).data_ptr(), int(bf16),
                                   master.data_ptr(), m.data_ptr(), v.data_ptr(),
                                   p16.data_ptr(), n, t[0], 1e-3, 0.9, 0.95, 1e-8, 0.1, 1.0, sp))
        return f

    timeit("adamw_flat_kernel<bf16>", adamw(True), 28 * n)
    timeit("adamw_flat_kernel<fp32>", adamw(False), 30 * n)
    timeit("upcast_scale", lambda: N.check(L.amsp_k_upcast_scale(
        g16.data_ptr(), out32.data_ptr(), n, 0.5, sp)), 6 * n)
    del g32
    srcs = [g16] + [torch.empty_like(g16).copy_(g16) for _ in range(3)]
    for W in (2, 4):
        ptrs = (C.c_void_p * W)(*[s.data_ptr() for s in srcs[:W]])
        timeit(f"rs_upcast_scale_kernel<{W}>", lambda ptrs=ptrs, W=W: N.check(
            L.amsp_k_rs_upcast_scale(ptrs, W, 0, out32.data_ptr(), n, 1.0 / W, sp)),
            (2 * W + 4) * n)
    for k in (1, 4):
        dst = [s.data_ptr() for s in srcs[:k]]
        ptrs = (C.c_void_p * k)(*dst)
        timeit(f"ag_downcast_kernel<{k}>", lambda ptrs=ptrs, k=k: N.check(
            L.amsp_k_ag_downcast(master.data_ptr(), n, ptrs, k, 0, sp)), (4 + 2 * k) * n)


if __name__ == "__main__":
    main()
