"""ctypes binding of oracle/amsp_oracle.c (test infrastructure only; see the
header of amsp_oracle.c — floating-point parity is "unpinned" by the
reference, which has no data plane)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_build" / "libamsp_oracle.so"


class Scalars(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("beta1", "one_minus_beta1", "beta2", "one_minus_beta2",
                                         "step_size", "inv_sqrt_bc2", "eps", "decay",
                                         "grad_scale")]


class Accum(C.Structure):
    _fields_ = [("micro_batches", C.c_int), ("staged", C.c_int), ("nblocks", C.c_int),
                ("block_of", C.c_int * 16)]


class Hyper(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("lr", "beta1", "beta2", "eps", "weight_decay")]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise ImportError(f"{LIB} missing: run __graft_entry__.build()")
        L = C.CDLL(str(LIB))
        u64p = C.POINTER(C.c_uint64)
        fp = C.POINTER(C.c_float)
        u16p = C.POINTER(C.c_uint16)
        L.amsp_o_set_threads.restype = C.c_int
        L.amsp_o_set_threads.argtypes = [C.c_int]
        L.amsp_o_grad_bf16.restype = C.c_uint16
        L.amsp_o_grad_bf16.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
        L.amsp_o_master_init.restype = C.c_float
        L.amsp_o_master_init.argtypes = [C.c_uint64, C.c_uint64]
        L.amsp_o_trajectory.argtypes = [u64p, C.c_size_t, C.c_uint64, C.c_int, C.c_int,
                                        C.POINTER(Hyper), fp, fp, fp, u16p]
        L.amsp_o_trajectory_range.argtypes = [C.c_uint64, C.c_size_t, C.c_uint64, C.c_int,
                                              C.c_int, C.POINTER(Hyper), fp, fp, fp, u16p]
        L.amsp_o_trajectory_acc.argtypes = [u64p, C.c_size_t, C.c_uint64, C.c_int, C.c_int,
                                            C.POINTER(Accum), C.POINTER(Hyper), fp, fp, fp,
                                            u16p]
        L.amsp_o_trajectory_range_acc.argtypes = [C.c_uint64, C.c_size_t, C.c_uint64, C.c_int,
                                                  C.c_int, C.POINTER(Accum), C.POINTER(Hyper),
                                                  fp, fp, fp, u16p]
        L.amsp_o_fill_grads_mb.argtypes = [u16p, C.c_uint64, C.c_size_t, C.c_uint64,
                                           C.c_uint32, C.c_uint32, C.c_uint32]
        L.amsp_o_reduced_grad.restype = C.c_float
        L.amsp_o_reduced_grad.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int,
                                          C.POINTER(Accum)]
        L.amsp_o_fill_grads.argtypes = [u16p, C.c_uint64, C.c_size_t, C.c_uint64, C.c_uint32,
                                        C.c_uint32]
        L.amsp_o_partition_greedy.argtypes = [u64p, C.c_int, C.c_int, C.POINTER(C.c_int),
                                              C.POINTER(C.c_int), u64p]
        L.amsp_o_adam_scalars.argtypes = [C.c_double] * 5 + [C.c_int, C.c_int,
                                                             C.POINTER(Scalars)]
        L.amsp_o_step.argtypes = [C.POINTER(u16p), C.c_int, u64p, u64p, u64p, C.c_int, fp, fp,
                                  fp, C.POINTER(u16p), C.c_int, C.POINTER(Scalars)]
        _lib = L
    return _lib


def use_all_threads() -> int:
    """Run the CPU step on every host thread (torchrun exports
    OMP_NUM_THREADS=1); returns the thread count in effect."""
    import os
    return lib().amsp_o_set_threads(os.cpu_count() or 1)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def hyper(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1) -> Hyper:
    return Hyper(lr, beta1, beta2, eps, weight_decay)


def mesh_blocks(dp, mesh, world: int) -> list:
    """block_of[rank] for the blocks of component `mesh` ((per_node, nodes))
    tiling the DP mesh `dp`, ranks node-major (rank = node*per_node + local),
    blocks numbered in order of their smallest rank. Restated from the
    paper's 2-level device mesh for the checker."""
    P, _ = dp
    a, b = mesh
    return [((r // P) // b) * (P // a) + (r % P) // a for r in range(world)]


def accum(micro_batches: int, sg: int, block_of) -> Accum:
    """Accumulation recipe: M micro-batches; s_g = 1 accumulates in place,
    s_g > 1 through the bf16 G shards of the blocks in `block_of`."""
    a = Accum()
    a.micro_batches = micro_batches
    a.staged = int(sg > 1)
    a.nblocks = max(block_of) + 1
    for r, blk in enumerate(block_of):
        a.block_of[r] = blk
    return a


def trajectory(index: np.ndarray, seed: int, steps: int, world: int, h: Hyper,
               acc: Accum | None = None):
    """(master, m, v, bf16 param) of the given flat indices after `steps`."""
    index = np.ascontiguousarray(index, dtype=np.uint64)
    n = index.size
    out = [np.empty(n, np.float32) for _ in range(3)] + [np.empty(n, np.uint16)]
    lib().amsp_o_trajectory_acc(_p(index, C.c_uint64), n, seed, steps, world,
                                C.byref(acc) if acc is not None else None, C.byref(h),
                                _p(out[0], C.c_float), _p(out[1], C.c_float),
                                _p(out[2], C.c_float), _p(out[3], C.c_uint16))
    return out


def trajectory_range(start: int, n: int, seed: int, steps: int, world: int, h: Hyper,
                     acc: Accum | None = None):
    out = [np.empty(n, np.float32) for _ in range(3)] + [np.empty(n, np.uint16)]
    lib().amsp_o_trajectory_range_acc(start, n, seed, steps, world,
                                      C.byref(acc) if acc is not None else None, C.byref(h),
                                      _p(out[0], C.c_float), _p(out[1], C.c_float),
                                      _p(out[2], C.c_float), _p(out[3], C.c_uint16))
    return out


def grads_mb(start: int, n: int, seed: int, step: int, micro_batch: int,
             rank: int) -> np.ndarray:
    out = np.empty(n, np.uint16)
    lib().amsp_o_fill_grads_mb(_p(out, C.c_uint16), start, n, seed, step, micro_batch, rank)
    return out


def reduced_grad(seed: int, step: int, index: int, world: int,
                 acc: Accum | None = None) -> float:
    return lib().amsp_o_reduced_grad(seed, step, index, world,
                                     C.byref(acc) if acc is not None else None)


def grads(start: int, n: int, seed: int, step: int, rank: int) -> np.ndarray:
    out = np.empty(n, np.uint16)
    lib().amsp_o_fill_grads(_p(out, C.c_uint16), start, n, seed, step, rank)
    return out


def master_init(seed: int, index: int) -> float:
    return lib().amsp_o_master_init(seed, index)


def partition_greedy(sizes, k):
    sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
    n = sizes.size
    order = np.empty(max(n, 1), np.int32)
    asg = np.empty(max(n, 1), np.int32)
    ss = np.empty(max(k, 1), np.uint64)
    rc = lib().amsp_o_partition_greedy(_p(sizes, C.c_uint64), n, k, _p(order, C.c_int),
                                       _p(asg, C.c_int), _p(ss, C.c_uint64))
    if rc:
        raise ValueError("oracle partition: bad input")
    return asg[:n].tolist(), ss[:k].tolist()


def scalars(step: int, world: int, h: Hyper) -> Scalars:
    s = Scalars()
    lib().amsp_o_adam_scalars(h.lr, h.beta1, h.beta2, h.eps, h.weight_decay, step, world,
                              C.byref(s))
    return s


def step(grad_bufs, segs, master, m, v, param_bufs, s: Scalars) -> None:
    """One CPU AMSP step over host arrays (the bench CPU baseline)."""
    u16p = C.POINTER(C.c_uint16)
    W = len(grad_bufs)
    gp = (u16p * W)(*[_p(g, C.c_uint16) for g in grad_bufs])
    dp = (u16p * len(param_bufs))(*[_p(p, C.c_uint16) for p in param_bufs])
    f = np.array([x[0] for x in segs], np.uint64)
    o = np.array([x[1] for x in segs], np.uint64)
    ln = np.array([x[2] for x in segs], np.uint64)
    lib().amsp_o_step(gp, W, _p(f, C.c_uint64), _p(o, C.c_uint64), _p(ln, C.c_uint64),
                      len(segs), _p(master, C.c_float), _p(m, C.c_float), _p(v, C.c_float),
                      dp, len(param_bufs), C.byref(s))
