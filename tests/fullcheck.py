"""Every-element parity at full model size, streamed in chunks.

The oracle's trajectory of an element depends only on its flat index
(oracle/amsp_oracle.c: counter-based gradients, per-element AdamW), so a
rank's whole P shard can be recomputed on the host in O(chunk) memory and
compared with the device buffers read back chunk by chunk. This is how the
BASELINE-sized configs (LLaMA-7B: 6.7e9 params, 108 GB of state; 13B
ZeRO-3) are checked bit-exactly without 100+ GB of host RAM.
"""
from __future__ import annotations

import bisect

import numpy as np

from oracle import cpu as O
from paper_2311_00257_b200.engine import DEFAULT_SEED, pshard_layout

CHUNK = 1 << 25


def check_engine(e, steps: int, world: int, chunk: int = CHUNK, log=print) -> list[str]:
    """Compare e's bf16 P shard and its fp32 master/m/v OS shard with the
    oracle after `steps` steps of `world` ranks. Returns mismatch messages
    (empty = bit-exact on every element)."""
    h = O.hyper()
    psegs, pn = pshard_layout(e.tensor_sizes, e.plan.sp(), e.info.p_position, 1, 0,
                              "contiguous")
    os_segs = sorted(e.segments()[0])  # (flat, os, len), by flat index
    os_starts = [f for f, _, _ in os_segs]
    bad: list[str] = []
    checked_p = checked_os = 0
    for f0, _, d0, ln in psegs:
        off = 0
        while off < ln:
            n = min(chunk, ln - off)
            a = f0 + off
            want = O.trajectory_range(a, n, DEFAULT_SEED, steps, world, h)
            got = e.read("params", d0 + off, n)
            if not np.array_equal(got, want[3]):
                i = int(np.argmax(got != want[3]))
                bad.append(f"params flat {a + i}: {got[i]:#06x} != {want[3][i]:#06x}")
            checked_p += n
            # owned OS segments overlapping [a, a+n)
            j = max(bisect.bisect_right(os_starts, a) - 1, 0)
            while j < len(os_segs) and os_segs[j][0] < a + n:
                sf, so, sl = os_segs[j]
                lo, hi = max(sf, a), min(sf + sl, a + n)
                if lo < hi:
                    for name, ref in zip(("master", "exp_avg", "exp_avg_sq"), want[:3]):
                        g = e.read(name, so + (lo - sf), hi - lo)
                        r = ref[lo - a:hi - a]
                        if not np.array_equal(g.view(np.uint32), r.view(np.uint32)):
                            i = int(np.argmax(g.view(np.uint32) != r.view(np.uint32)))
                            bad.append(f"{name} flat {lo + i}: {g[i]!r} != {r[i]!r}")
                    checked_os += hi - lo
                j += 1
            off += n
            if len(bad) > 8:
                return bad
    if checked_p != pn:
        bad.append(f"checked {checked_p} of {pn} P-shard elements")
    if checked_os != e.info.owned:
        bad.append(f"checked {checked_os} of {e.info.owned} owned elements")
    log(f"fullcheck: {checked_p} params + {checked_os} x 3 optimizer-state elements compared")
    return bad
