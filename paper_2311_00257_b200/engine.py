"""AMSP step engine (the B200 data plane) over the C-ABI.

One Engine per GPU / process. The engine owns the rank's model-state
buffers; peers are connected by exchanging cudaIpc handles (64 bytes per
rank) through any all-gather — torch.distributed is used here purely as
plumbing. There is no CPU path: every method launches sm_100a kernels in
libamsp.so or raises.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .shardplan import DeviceMesh, ModelSpec, ShardingPlan, llama_tensors

LAYOUTS = {"greedy": 0, "contiguous": 1}
BUFFERS = {"grads": (0, np.uint16), "params": (1, np.uint16), "master": (2, np.float32),
           "exp_avg": (3, np.float32), "exp_avg_sq": (4, np.float32),
           "slot0": (5, np.uint16), "slot1": (6, np.uint16), "acc": (7, np.uint16)}
DEFAULT_SEED = 0x414D5350  # "AMSP"


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)  # torch.cuda.Stream


class Engine:
    def __init__(self, tensors: Sequence[int] | ModelSpec, plan: ShardingPlan,
                 dp_mesh: DeviceMesh, rank: int = 0, device: int = 0,
                 layout: str = "greedy", lr: float = 1e-3, betas=(0.9, 0.95),
                 eps: float = 1e-8, weight_decay: float = 0.1, seed: int = DEFAULT_SEED,
                 skip_gathers: bool = False, micro_batches: int = 1, grad_ring: int = 0):
        if isinstance(tensors, ModelSpec):
            tensors = llama_tensors(tensors)
        self.tensor_sizes = [int(t) for t in tensors]
        self.plan, self.dp_mesh, self.rank = plan, dp_mesh, rank
        self.hyper = dict(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps,
                          weight_decay=weight_decay)
        self.seed = seed
        self.layout = layout
        arr = (C.c_uint64 * len(self.tensor_sizes))(*self.tensor_sizes)
        cfg = N.EngineConfig(C.cast(arr, C.POINTER(C.c_uint64)), len(self.tensor_sizes),
                             plan._c(), dp_mesh._c(), rank, device, LAYOUTS[layout], lr,
                             betas[0], betas[1], eps, weight_decay, seed, int(skip_gathers),
                             int(micro_batches), int(grad_ring))
        self._h = C.c_void_p()
        N.check(N.lib().amsp_engine_create(C.byref(cfg), C.byref(self._h)))
        self.info = self._info()

    def _info(self) -> N.EngineInfo:
        info = N.EngineInfo()
        N.check(N.lib().amsp_engine_info(self._h, C.byref(info)))
        return info

    @property
    def world(self) -> int:
        return self.info.world

    # ---------------------------------------------------------- peers
    def export_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        N.check(N.lib().amsp_engine_export_handle(self._h, buf))
        return bytes(buf)

    def import_handles(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        N.check(N.lib().amsp_engine_import_handles(self._h, blob, len(handles)))

    def connect(self, group=None) -> None:
        """Exchange IPC handles with every DP rank via torch.distributed."""
        if self.world == 1:
            return
        self.import_handles(exchange_handles(self.export_handle(), self.world, group))

    # ---------------------------------------------------------- work
    def init_state(self, stream=None) -> None:
        N.check(N.lib().amsp_engine_init_state(self._h, _stream_ptr(stream)))

    def synth_grads(self, step: int, stream=None, mb: int = 0) -> None:
        """Synthetic gradient of micro-batch `mb` of `step` (s_g = 1 and
        mb > 0: accumulated into the gradient buffer in place)."""
        N.check(N.lib().amsp_engine_synth_grads_mb(self._h, step, mb, _stream_ptr(stream)))

    def accumulate(self, step: int, mb: int, stream=None) -> None:
        """Micro-batch mb < M-1 is in every rank's gradient buffer: fold it
        into the G-shard accumulators (s_g > 1; a no-op for s_g = 1)."""
        N.check(N.lib().amsp_engine_accumulate(self._h, step, mb, _stream_ptr(stream)))

    def micro_step(self, step: int, stream=None) -> None:
        """One whole step of M micro-batches with synthetic gradients: for
        every micro-batch, synthesize it, then accumulate (mb < M-1) or run
        the optimizer step (the last)."""
        M = self.info.micro_batches
        for mb in range(M):
            self.synth_grads(step, stream, mb)
            if mb + 1 < M:
                self.accumulate(step, mb, stream)
        self.step(step, stream)

    def step(self, step: int, stream=None) -> None:
        N.check(N.lib().amsp_engine_step(self._h, step, _stream_ptr(stream)))

    def step_host(self, step: int, host_grads_ptr: int, stream=None) -> np.ndarray:
        stats = (C.c_float * 2)()
        N.check(N.lib().amsp_engine_step_host(self._h, step, C.c_void_p(host_grads_ptr),
                                              stats, _stream_ptr(stream)))
        return np.array(stats, dtype=np.float32)

    def stats(self) -> np.ndarray:
        s = (C.c_float * 2)()
        N.check(N.lib().amsp_engine_stats(self._h, s))
        return np.array(s, dtype=np.float32)

    def read(self, which: str, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
        idx, dt = BUFFERS[which]
        total = {0: self.info.total_params, 1: self.info.param_elems,
                 7: self.info.acc_elems}.get(idx, self.info.owned if idx < 5
                                             else self.info.slot_elems)
        count = total - offset if count is None else count
        out = np.empty(count, dtype=dt)
        N.check(N.lib().amsp_engine_read(self._h, idx, offset, count,
                                         out.ctypes.data_as(C.c_void_p)))
        return out

    def write(self, which: str, data: np.ndarray, offset: int = 0) -> None:
        idx, dt = BUFFERS[which]
        data = np.ascontiguousarray(data, dtype=dt)
        N.check(N.lib().amsp_engine_write(self._h, idx, offset, data.size,
                                          data.ctypes.data_as(C.c_void_p)))

    def launch_count(self) -> int:
        n = C.c_uint64()
        N.check(N.lib().amsp_engine_launch_count(self._h, C.byref(n)))
        return n.value

    def unit(self, u: int):
        """(first_tensor, n_tensors, elems) of all-gather unit u (s_p > 1)."""
        f, n, el = C.c_int(), C.c_int(), C.c_uint64()
        N.check(N.lib().amsp_engine_unit(self._h, u, C.byref(f), C.byref(n), C.byref(el)))
        return f.value, n.value, el.value

    def gather(self, unit: int, slot: int = 0, stream=None, secondary: bool = False) -> None:
        """All-gather of one unit into slot `slot`, from the P shards, or with
        `secondary` from the ZeRO++ secondary group's slices."""
        fn = N.lib().amsp_engine_gather_secondary if secondary else N.lib().amsp_engine_gather
        N.check(fn(self._h, unit, slot, _stream_ptr(stream)))

    def tune(self, variant: int = 0, grid: int = 0) -> None:
        N.check(N.lib().amsp_engine_tune(self._h, variant, grid))
        self.info = self._info()

    def tune_gather(self, mode) -> None:
        """All-gather implementation of engine.step / gather(): an SM-kernel
        grid (int > 0), "sm" (default grid), "dma" (copy engines), "tma"
        (bulk-copy kernel, pulls) or "push" (the step's passes store each
        rank's slice into its peers' slots; a single gather() still pulls)."""
        grid = {"sm": 0, "dma": -1, "tma": -2, "push": -3}.get(mode, mode)
        N.check(N.lib().amsp_engine_tune_gather(self._h, int(grid)))

    def time_kernel(self, enable: bool = True) -> None:
        N.check(N.lib().amsp_engine_time_kernel(self._h, int(enable)))

    def kernel_ms(self):
        """(summed fused-kernel ms, launches) since time_kernel(True)."""
        ms, n = C.c_double(), C.c_int()
        N.check(N.lib().amsp_engine_kernel_ms(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def accum_ms(self):
        """(summed micro-batch accumulation kernel ms, launches) since time_kernel(True)."""
        ms, n = C.c_double(), C.c_int()
        N.check(N.lib().amsp_engine_accum_ms(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def nvlink_probe(self, nbytes: int = 1 << 32, pattern: str = "all", iters: int = 5):
        """This rank's NVLink ingress in GB/s pulling `nbytes` from its peers
        (pattern "ring": all from rank+1; "all": an equal share from every
        peer). Collective: every rank must call it."""
        ms = C.c_double()
        N.check(N.lib().amsp_engine_nvlink_probe(self._h, nbytes, {"ring": 0, "all": 1}[pattern],
                                                 iters, C.byref(ms)))
        per = (nbytes // (1 if pattern == "ring" else self.world - 1)) // 16 * 16
        moved = min(per, 2 * self.info.grad_elems // 16 * 16) * (
            1 if pattern == "ring" else self.world - 1)
        return moved / (ms.value * 1e-3) / 1e9

    def gather_ms(self):
        """(summed all-gather-phase ms, steps) since time_kernel(True)."""
        ms, n = C.c_double(), C.c_int()
        N.check(N.lib().amsp_engine_gather_ms(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def segments(self):
        """(flat, os, len) triples of this rank's optimizer-state shard."""
        return self.shard_layout()[0], self.info.owned

    def shard_layout(self):
        """([(flat, os, dst, len)], owned) of this rank's optimizer-state shard."""
        segs, owned = pshard_layout(self.tensor_sizes, self.plan.sp(), self.info.p_position,
                                    self.info.os_group_size, self._k_position(), self.layout)
        return [(f, o, ln) for f, o, d, ln in segs], segs

    def _k_position(self):
        # index of this rank among its OS block's ranks with the same P position
        dp, plan = self.dp_mesh, self.plan
        _, _, members = mesh_group(dp, plan.os, self.rank)
        mine = mesh_group(dp, plan.p, self.rank)[1]
        same = [m for m in members if mesh_group(dp, plan.p, m)[1] == mine]
        return same.index(self.rank)

    def close(self) -> None:
        if self._h:
            N.lib().amsp_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Scheduler:
    """Overlap scheduler over an Engine (amsp_sched_*): replays the reference
    event graph for `model` / the engine's plan on 3 CUDA streams."""

    def __init__(self, engine: Engine, model: ModelSpec, profile, cost=None, sim=None,
                 comm_ctas: int = 0, compute_ctas: int = 0, time_scale: float = 1.0,
                 optimizer_overlap: bool = True, compute: str = "standin", tokens: int = 0,
                 gemm_sm_margin: int = 0, gather: str = "sm", bc: str = "auto",
                 optimizer_variant: int = 0, reduce: str = "sm", grad_source: str = "caller"):
        from .shardplan import CostConfig, SimConfig
        cost = cost or CostConfig()
        sim = sim or SimConfig()
        m, self._keep = model._c()
        k = model.modules_per_layer
        tabs = []

        def arr(v):
            if v is None:
                return None
            a = (C.c_double * k)(*v)
            tabs.append(a)
            return C.cast(a, C.POINTER(C.c_double))

        sc = N.SimConfig(SimConfig.TIERS.index(sim.overlap_tier), int(sim.recompute),
                         sim.comm_streams, 1 if sim.fwd_times is not None else 0,
                         sim.peak_flops_per_gpu, sim.compute_efficiency, arr(sim.fwd_times),
                         arr(sim.bwd_grad_weight_times), arr(sim.bwd_grad_input_times),
                         sim.head_fwd_time, sim.head_bwd_time)
        cfg = N.SchedConfig(m, cost._c(), sc, comm_ctas, compute_ctas, time_scale,
                            int(optimizer_overlap), {"standin": 0, "gemm": 1}[compute], tokens,
                            gemm_sm_margin, {"sm": 0, "dma": 1, "tma": 2}[gather],
                            {"auto": 0, "push": 1}[bc], optimizer_variant,
                            {"sm": 0, "dma": 1}[reduce], {"caller": 0, "synth": 1}[grad_source])
        self.engine = engine
        self._h = C.c_void_p()
        N.check(N.lib().amsp_sched_create(engine._h, C.byref(cfg), profile._h, C.byref(self._h)))
        self.info = N.SchedInfo()
        N.check(N.lib().amsp_sched_info(self._h, C.byref(self.info)))

    def step(self, step: int, stream=None, with_comm=True) -> None:
        """with_comm: True = full step, False = compute only, "optimizer" =
        compute + local optimizer work without communication (timing)."""
        mode = 2 if with_comm == "optimizer" else int(bool(with_comm))
        N.check(N.lib().amsp_sched_step(self._h, step, _stream_ptr(stream), mode))

    def barrier_owner(self, barrier_id: int):
        """(event index, role, micro-batch) of the graph event using a barrier
        id (diagnostics of a barrier timeout; amsp_sched_barrier_owner)."""
        ev, role, mb = C.c_int(), C.c_int(), C.c_int()
        N.check(N.lib().amsp_sched_barrier_owner(self._h, barrier_id, C.byref(ev),
                                                 C.byref(role), C.byref(mb)))
        roles = ["pre-reduce", "optimizer", "release", "head accumulation", "head release",
                 "end of step A", "end of step B", "flush"]
        return ev.value, roles[role.value], mb.value

    def flush(self, stream=None) -> None:
        """Mirrored broadcast (info.mirrored_bc): pull the other owners'
        updated parameters after the last step (every rank calls it)."""
        N.check(N.lib().amsp_sched_flush(self._h, _stream_ptr(stream)))

    def enable_trace(self, on: bool = True) -> None:
        N.check(N.lib().amsp_sched_enable_trace(self._h, int(on)))

    def trace(self):
        """(measured TEF JSON of the last traced step, its span in ms)."""
        need, ms = C.c_size_t(), C.c_double()
        N.check(N.lib().amsp_sched_trace(self._h, None, 0, C.byref(need), C.byref(ms)))
        buf = C.create_string_buffer(need.value + 1)
        N.check(N.lib().amsp_sched_trace(self._h, buf, need.value + 1, None, None))
        return buf.value.decode(), ms.value

    def predicted_trace(self) -> str:
        need = C.c_size_t()
        N.check(N.lib().amsp_sched_predicted_trace(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value + 1)
        N.check(N.lib().amsp_sched_predicted_trace(self._h, buf, need.value + 1, None))
        return buf.value.decode()

    def close(self) -> None:
        if self._h:
            N.lib().amsp_sched_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def b200_profile(world_max: int = 8):
    """Synthetic alpha-beta profile at the measured B200 NVLink rates
    (680 GB/s per direction for a plain P2P copy, 5 us latency) for every
    single-node mesh up to world_max GPUs — the planner's input when no
    measured CSV is supplied."""
    from .shardplan import BandwidthProfile
    meshes = [DeviceMesh(a, b) for a in range(1, world_max + 1) for b in (1, 2, 4, 8)]
    return BandwidthProfile.synthetic((5e-6, 680e9), (10e-6, 50e9), meshes,
                                      [1 << k for k in range(10, 36)])


def exchange_handles(handle: bytes, world: int, group=None) -> list:
    """All-gather every rank's 64-byte cudaIpc handle, in rank order."""
    import torch.distributed as dist
    if len(handle) != 64:
        raise ValueError("IPC handles are 64 bytes")
    handles = [None] * world
    dist.all_gather_object(handles, handle, group=group)
    if any(not isinstance(h, bytes) or len(h) != 64 for h in handles):
        raise RuntimeError("malformed IPC handle received from a peer")
    return handles


def link_local(engines: Sequence[Engine], sync: bool = False) -> None:
    """Emulate one DP group on a single GPU (tests/smoke): engines must be
    ranks 0..n-1 created on the same device. sync=False: steps run one after
    another on one stream without cross-GPU barriers. sync=True: every
    engine keeps its own stream and the real barrier kernels / release
    fences order the ranks, as across GPUs (amsp_engine_link_local_sync)."""
    arr = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
    fn = N.lib().amsp_engine_link_local_sync if sync else N.lib().amsp_engine_link_local
    N.check(fn(arr, len(engines)))
    for e in engines:
        e._linked = engines  # keep peers alive while linked


def layout_segments(tensor_sizes: Sequence[int], shard_count: int, shard: int,
                    layout: str = "greedy"):
    n = len(tensor_sizes)
    arr = (C.c_uint64 * max(n, 1))(*tensor_sizes)
    nseg, owned = C.c_int(), C.c_uint64()
    N.check(N.lib().amsp_layout_segments(arr, n, shard_count, shard, LAYOUTS[layout], None,
                                         None, None, 0, C.byref(nseg), C.byref(owned)))
    k = max(nseg.value, 1)
    f, o, ln = (C.c_uint64 * k)(), (C.c_uint64 * k)(), (C.c_uint64 * k)()
    N.check(N.lib().amsp_layout_segments(arr, n, shard_count, shard, LAYOUTS[layout], f, o,
                                         ln, k, C.byref(nseg), C.byref(owned)))
    return [(f[i], o[i], ln[i]) for i in range(nseg.value)], owned.value


def pshard_layout(tensor_sizes: Sequence[int], sp: int, p_pos: int, k: int, os_pos: int,
                  layout: str = "greedy"):
    """([(flat, os, dst, len)], owned) — see amsp_pshard_layout."""
    n = len(tensor_sizes)
    arr = (C.c_uint64 * max(n, 1))(*tensor_sizes)
    nseg, owned = C.c_int(), C.c_uint64()
    N.check(N.lib().amsp_pshard_layout(arr, n, sp, p_pos, k, os_pos, LAYOUTS[layout], None,
                                       None, None, None, 0, C.byref(nseg), C.byref(owned)))
    m = max(nseg.value, 1)
    f, o, d, ln = [(C.c_uint64 * m)() for _ in range(4)]
    N.check(N.lib().amsp_pshard_layout(arr, n, sp, p_pos, k, os_pos, LAYOUTS[layout], f, o, d,
                                       ln, m, C.byref(nseg), C.byref(owned)))
    return [(f[i], o[i], d[i], ln[i]) for i in range(nseg.value)], owned.value


def mesh_group(dp: DeviceMesh, mesh: DeviceMesh, rank: int):
    blk, pos, n = C.c_int(), C.c_int(), C.c_int()
    mem = (C.c_int * 64)()
    N.check(N.lib().amsp_mesh_group(dp._c(), mesh._c(), rank, C.byref(blk), C.byref(pos), mem,
                                    64, C.byref(n)))
    return blk.value, pos.value, list(mem)[:n.value]
