#!/usr/bin/env python
"""SASS evidence for the default TMA kernels (run here, no GPU): per kernel,
the counts of bulk-copy (UBLKCP), mbarrier (SYNCS), 128-bit global load /
store and peer-store instructions, plus the first bulk-copy / mbarrier lines.

  python tools/sass_excerpt.py [libamsp.so] > profiles/r02_sass_tma_excerpt.txt
"""
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(sys.argv[1] if len(sys.argv) > 1 else
           Path(__file__).resolve().parents[1] / "paper_2311_00257_b200" / "libamsp.so")
KERNELS = {  # engine_impl.h retune(): the auto variant per W
    "fused_step_tma_kernelILi1ELi3ELi2ELb0E": "W=1 default (variant 5: 3-stage ring, 2 CTAs/SM)",
    "fused_step_tma_kernelILi2ELi5ELi1ELb1E": "W=2 default (variant 11: 5 stages + bulk drain)",
    "fused_step_tma_kernelILi4ELi4ELi2ELb0E": "W=4 default (variant 10: 4-stage ring)",
    "fused_step_tma_kernelILi8ELi2ELi2ELb0E": "W=8 default (variant 5: 2-stage ring, 2 CTAs/SM)",
    "gather_tma_kernel": "all-gather (s_p > 1) default",
}
text = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True,
                      check=True).stdout
funcs = re.split(r"\n\s*Function : ", text)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    key = next((k for k in KERNELS if k in name), None)
    if not key:
        continue
    body = f.split("\n", 1)[1]
    ins = [ln for ln in body.splitlines() if re.search(r"/\*[0-9a-f]{4,}\*/", ln)]
    count = lambda pat: sum(1 for ln in ins if re.search(pat, ln))  # noqa: E731
    print(f"== {name}\n   {KERNELS[key]}")
    print(f"   instructions {len(ins)}: UBLKCP {count(r'UBLKCP')}, SYNCS {count(r'SYNCS')}, "
          f"LDG.E.128 {count(r'LDG\\.E\\.128')}, STG.E.128 {count(r'STG\\.E\\.128')}, "
          f"LDS.128 {count(r'LDS\\.128')}, MEMBAR {count(r'MEMBAR')}")
    shown = 0
    for ln in ins:
        if re.search(r"UBLKCP|SYNCS", ln) and shown < 8:
            print("   " + re.sub(r"\s+", " ", ln.strip())[:120])
            shown += 1
    print()
