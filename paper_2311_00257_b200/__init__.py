"""B200-native AMSP (arXiv 2311.00257) model-state pipeline.

- `shardplan`: drop-in mirror of the reference planner API (validate_plan,
  presets, cost model, solver, overlap simulator), backed by the C++
  implementation in csrc/plan/ through the C-ABI (include/amsp_c.h).
- `engine`: the sm_100a data plane — fused gradient reduce + sharded AdamW +
  parameter gather over NVLink peer memory.
"""
from . import shardplan  # noqa: F401
from ._native import lib  # noqa: F401

__all__ = ["shardplan", "lib"]
