"""Python mirror of the reference `shardplan` planner API over the C-ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/shardplan/*.hpp): value types for meshes,
clusters, models and plans; `validate_plan` returns violations instead of
raising; `preset` raises InfeasibleError; `solve` raises NoFeasiblePlanError
carrying the closest candidate. Every call goes through libamsp.so (the C++
drop-in implementation in csrc/plan/), never through Python arithmetic.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import _native as N

Error = N.InvalidConfig


class InfeasibleError(N.Infeasible):
    pass


class NoFeasiblePlanError(N.Infeasible):
    def __init__(self, code: int, msg: str, closest: "PlanResult"):
        super().__init__(code, msg)
        self._closest = closest

    def closest(self) -> "PlanResult":
        return self._closest


@dataclass(frozen=True, order=True)
class DeviceMesh:
    per_node: int = 1
    nodes: int = 1

    def size(self) -> int:
        return self.per_node * self.nodes

    def __str__(self) -> str:
        return f"{self.per_node}x{self.nodes}"

    def _c(self) -> N.Mesh:
        return N.Mesh(self.per_node, self.nodes)

    @staticmethod
    def _from(m: N.Mesh) -> "DeviceMesh":
        return DeviceMesh(m.per_node, m.nodes)


@dataclass
class Topology:
    leaf_count: int = 1
    nodes_per_leaf: int = 1
    inter_leaf_penalty: float = 1.0


@dataclass
class ClusterSpec:
    gpus_per_node: int = 8
    node_count: int = 1
    gpu_memory_capacity: int = 0
    dp_mesh: DeviceMesh = field(default_factory=DeviceMesh)
    topology: Topology = field(default_factory=Topology)

    def gpu_count(self) -> int:
        return self.gpus_per_node * self.node_count

    def _c(self) -> N.Cluster:
        return N.Cluster(self.gpus_per_node, self.node_count, self.gpu_memory_capacity,
                         self.dp_mesh._c(), self.topology.leaf_count,
                         self.topology.nodes_per_leaf, self.topology.inter_leaf_penalty)


@dataclass
class ModelSpec:
    total_params: int = 0
    layer_count: int = 1
    modules_per_layer: int = 1
    module_params: Sequence[int] = ()
    hidden: int = 1
    seq_len: int = 1
    micro_batch: int = 1
    micro_batch_count: int = 1
    vocab: int = 1
    bytes_per_param: int = 2
    bytes_per_grad: int = 2
    bytes_per_os_per_param: int = 12

    def layer_template_params(self) -> int:
        return sum(self.module_params)

    def _c(self):
        arr = (C.c_uint64 * max(1, len(self.module_params)))(*self.module_params)
        m = N.Model(self.total_params, self.layer_count, self.modules_per_layer,
                    C.cast(arr, C.POINTER(C.c_uint64)), self.hidden, self.seq_len,
                    self.micro_batch, self.micro_batch_count, self.vocab,
                    self.bytes_per_param, self.bytes_per_grad, self.bytes_per_os_per_param)
        return m, arr  # keep arr alive


@dataclass(frozen=True)
class ShardingPlan:
    p: DeviceMesh = DeviceMesh()
    g: DeviceMesh = DeviceMesh()
    os: DeviceMesh = DeviceMesh()
    secondary_params: Optional[DeviceMesh] = None

    def sp(self) -> int:
        return self.p.size()

    def sg(self) -> int:
        return self.g.size()

    def sos(self) -> int:
        return self.os.size()

    def lex_key(self):
        return (self.p.per_node, self.p.nodes, self.g.per_node, self.g.nodes,
                self.os.per_node, self.os.nodes)

    def __str__(self) -> str:
        s = f"p={self.p},g={self.g},os={self.os}"
        return s + (f",p2={self.secondary_params}" if self.secondary_params else "")

    def _c(self) -> N.Plan:
        sec = self.secondary_params
        return N.Plan(self.p._c(), self.g._c(), self.os._c(), 1 if sec else 0,
                      (sec or DeviceMesh())._c())

    @staticmethod
    def _from(p: N.Plan) -> "ShardingPlan":
        return ShardingPlan(DeviceMesh._from(p.p), DeviceMesh._from(p.g),
                            DeviceMesh._from(p.os),
                            DeviceMesh._from(p.secondary) if p.has_secondary else None)


@dataclass
class CostConfig:
    bucket_size: int = 1 << 27
    activation_mode: int = 0  # 0 None, 1 FullRecompute
    activation_coeff_full: float = 34.0
    activation_coeff_recompute: float = 2.0
    tmp_in_flight_buckets: int = 2
    tmp_include_gather_buffer: bool = True
    exact_residual_buckets: bool = False
    flops_coeff_param: float = 6.0
    flops_coeff_attn: float = 12.0

    def _c(self) -> N.CostConfig:
        return N.CostConfig(self.bucket_size, self.activation_mode,
                            self.activation_coeff_full, self.activation_coeff_recompute,
                            self.tmp_in_flight_buckets, int(self.tmp_include_gather_buffer),
                            int(self.exact_residual_buckets), self.flops_coeff_param,
                            self.flops_coeff_attn)


@dataclass
class SimConfig:
    overlap_tier: str = "ag_rs_ar_bc"
    recompute: bool = False
    comm_streams: int = 2
    peak_flops_per_gpu: float = 312e12
    compute_efficiency: float = 0.6
    fwd_times: Optional[Sequence[float]] = None
    bwd_grad_weight_times: Optional[Sequence[float]] = None
    bwd_grad_input_times: Optional[Sequence[float]] = None
    head_fwd_time: float = 0.0
    head_bwd_time: float = 0.0

    TIERS = ("none", "ag_rs", "ag_rs_ar", "ag_rs_ar_bc")


@dataclass
class TimeBreakdown:
    t_p: float
    t_g: float
    t_os_allreduce: float
    t_os_broadcast: float
    total: float


@dataclass
class MemoryBreakdown:
    d_params: float
    d_grads: float
    d_os: float
    d_modelstate: float
    d_activation: float
    d_tmp: float
    d_total: float


@dataclass
class PlanResult:
    plan: ShardingPlan
    time: TimeBreakdown
    memory: MemoryBreakdown
    feasible: bool
    rank: int

    @staticmethod
    def _from(r: N.PlanResult) -> "PlanResult":
        return PlanResult(ShardingPlan._from(r.plan),
                          TimeBreakdown(*(getattr(r.time, f) for f, _ in N.TimeBreakdown._fields_)),
                          MemoryBreakdown(*(getattr(r.memory, f) for f, _ in
                                            N.MemoryBreakdown._fields_)),
                          bool(r.feasible), r.rank)


@dataclass
class SearchReport:
    best: PlanResult
    candidates_evaluated: int
    candidates_filtered: int
    all_results: Optional[list]


@dataclass
class Violation:
    constraint: str
    detail: str


@dataclass
class ValidationResult:
    violations: list

    def ok(self) -> bool:
        return not self.violations


@dataclass
class SimResult:
    step_time: float
    compute_idle: float
    n_events: int
    trace: str


COLLECTIVES = {"allgather": 0, "reducescatter": 1, "allreduce": 2, "broadcast": 3}
PRESET_NAMES = ("ZeRO-1", "ZeRO-3", "MiCS", "ZeRO++", "AMSP-7B", "AMSP-13B", "AMSP-30B")


def preset_names():
    return list(PRESET_NAMES)


def _call(fn, *args):
    N.check(fn(*args))


class BandwidthProfile:
    """Opaque handle to shardplan::BandwidthProfile."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            N.lib().amsp_profile_free(h)
            self._h = C.c_void_p()

    @staticmethod
    def synthetic(ab_intra, ab_inter, meshes, sizes) -> "BandwidthProfile":
        ms = (N.Mesh * len(meshes))(*[m._c() for m in meshes])
        sz = (C.c_uint64 * len(sizes))(*sizes)
        out = C.c_void_p()
        _call(N.lib().amsp_profile_synthetic, ab_intra[0], ab_intra[1], ab_inter[0],
              ab_inter[1], ms, len(meshes), sz, len(sizes), C.byref(out))
        return BandwidthProfile(out.value)

    @staticmethod
    def from_csv(text: str) -> "BandwidthProfile":
        out = C.c_void_p()
        _call(N.lib().amsp_profile_from_csv, text.encode(), C.byref(out))
        return BandwidthProfile(out.value)

    @staticmethod
    def from_json(text: str) -> "BandwidthProfile":
        out = C.c_void_p()
        _call(N.lib().amsp_profile_from_json, text.encode(), C.byref(out))
        return BandwidthProfile(out.value)

    @staticmethod
    def load(path: str) -> "BandwidthProfile":
        out = C.c_void_p()
        _call(N.lib().amsp_profile_load, str(path).encode(), C.byref(out))
        return BandwidthProfile(out.value)

    def to_canonical_json(self) -> str:
        need = C.c_size_t()
        _call(N.lib().amsp_profile_to_json, self._h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value + 1)
        _call(N.lib().amsp_profile_to_json, self._h, buf, need.value + 1, C.byref(need))
        return buf.value.decode()

    def collective_time(self, kind: str, size_bytes: int, mesh: DeviceMesh) -> float:
        out = C.c_double()
        _call(N.lib().amsp_collective_time, self._h, COLLECTIVES[kind], size_bytes,
              mesh._c(), C.byref(out))
        return out.value


def ring_time(kind: str, size_bytes: float, participants: int, alpha: float,
              link_bandwidth: float) -> float:
    out = C.c_double()
    _call(N.lib().amsp_ring_time, COLLECTIVES[kind], size_bytes, participants, alpha,
          link_bandwidth, C.byref(out))
    return out.value


def validate_plan(plan: ShardingPlan, cluster: ClusterSpec) -> ValidationResult:
    n = C.c_int()
    buf = C.create_string_buffer(1 << 14)
    p, c = plan._c(), cluster._c()
    _call(N.lib().amsp_validate_plan, C.byref(p), C.byref(c), C.byref(n), buf, len(buf))
    vs = []
    for line in buf.value.decode().splitlines():
        k, _, d = line.partition(":")
        vs.append(Violation(k, d))
    return ValidationResult(vs)


def preset(name: str, cluster: ClusterSpec) -> ShardingPlan:
    out = N.Plan()
    c = cluster._c()
    code = N.lib().amsp_preset(name.encode(), C.byref(c), C.byref(out))
    if code == N.AMSP_EINFEASIBLE:
        raise InfeasibleError(code, N.lib().amsp_last_error().decode())
    N.check(code)
    return ShardingPlan._from(out)


def memory_breakdown(model: ModelSpec, plan: ShardingPlan,
                     cfg: CostConfig = CostConfig()) -> MemoryBreakdown:
    m, _keep = model._c()
    p, c, out = plan._c(), cfg._c(), N.MemoryBreakdown()
    _call(N.lib().amsp_memory_breakdown, C.byref(m), C.byref(p), C.byref(c), C.byref(out))
    return MemoryBreakdown(*(getattr(out, f) for f, _ in N.MemoryBreakdown._fields_))


def total_comm_time(model: ModelSpec, cluster: ClusterSpec, plan: ShardingPlan,
                    profile: BandwidthProfile, cfg: CostConfig = CostConfig()) -> TimeBreakdown:
    m, _keep = model._c()
    cl, p, c, out = cluster._c(), plan._c(), cfg._c(), N.TimeBreakdown()
    _call(N.lib().amsp_total_comm_time, C.byref(m), C.byref(cl), C.byref(p), profile._h,
          C.byref(c), C.byref(out))
    return TimeBreakdown(*(getattr(out, f) for f, _ in N.TimeBreakdown._fields_))


def grad_bucket_count(model: ModelSpec, plan: ShardingPlan,
                      cfg: CostConfig = CostConfig()) -> int:
    m, _keep = model._c()
    p, c, out = plan._c(), cfg._c(), C.c_uint64()
    _call(N.lib().amsp_grad_bucket_count, C.byref(m), C.byref(p), C.byref(c), C.byref(out))
    return out.value


def partition_tensors_greedy(sizes: Sequence[int], shard_count: int):
    n = len(sizes)
    arr = (C.c_uint64 * max(n, 1))(*sizes)
    asg = (C.c_int * max(n, 1))()
    ss = (C.c_uint64 * max(shard_count, 1))()
    _call(N.lib().amsp_partition_greedy, arr, n, shard_count, asg, ss)
    return list(asg)[:n], list(ss)[:shard_count]


def enumerate_candidates(cluster: ClusterSpec) -> list:
    c = cluster._c()
    n = C.c_int()
    _call(N.lib().amsp_enumerate_candidates, C.byref(c), None, 0, C.byref(n))
    arr = (N.Plan * max(n.value, 1))()
    _call(N.lib().amsp_enumerate_candidates, C.byref(c), arr, n.value, C.byref(n))
    return [ShardingPlan._from(arr[i]) for i in range(n.value)]


def solve(model: ModelSpec, cluster: ClusterSpec, profile: BandwidthProfile,
          cfg: CostConfig = CostConfig(), keep_all_results: bool = False) -> SearchReport:
    m, _keep = model._c()
    cl, c = cluster._c(), cfg._c()
    best, ev, fi, n_all = N.PlanResult(), C.c_uint64(), C.c_uint64(), C.c_int()
    cap = 4096 if keep_all_results else 0
    allr = (N.PlanResult * max(cap, 1))()
    code = N.lib().amsp_solve(C.byref(m), C.byref(cl), profile._h, C.byref(c), C.byref(best),
                              C.byref(ev), C.byref(fi), allr if cap else None, cap,
                              C.byref(n_all) if cap else None)
    if code == N.AMSP_EINFEASIBLE:
        raise NoFeasiblePlanError(code, N.lib().amsp_last_error().decode(),
                                  PlanResult._from(best))
    N.check(code)
    all_results = [PlanResult._from(allr[i]) for i in range(n_all.value)] if cap else None
    return SearchReport(PlanResult._from(best), ev.value, fi.value, all_results)


# ----------------------------------------------------------- B200 roofline
# Not part of the reference API: the engine's step roofline and the solver
# that ranks the reference's candidates by it (engine/roofline.h).

B200_HBM_BW = 6524e9     # MEASURED_PEAKS.json copy bandwidth (bytes/s)
B200_NVLINK_BW = 770e9   # measured peer copy per direction (B200_PROFILING.md)
LAYOUTS = {"greedy": 0, "contiguous": 1}


@dataclass
class StepRoofline:
    owned: int
    hbm_bytes: int
    nvlink_in_bytes: int
    nvlink_out_bytes: int
    t_hbm: float
    t_nvlink: float
    t_step: float

    @staticmethod
    def _from(r: N.StepRoofline) -> "StepRoofline":
        return StepRoofline(r.owned, r.hbm_bytes, r.nvlink_in_bytes, r.nvlink_out_bytes,
                            r.t_hbm, r.t_nvlink, r.t_step)


def model_tensors(model: ModelSpec) -> list:
    m, _keep = model._c()
    n = C.c_int()
    _call(N.lib().amsp_model_tensors, C.byref(m), None, 0, C.byref(n))
    arr = (C.c_uint64 * max(n.value, 1))()
    _call(N.lib().amsp_model_tensors, C.byref(m), arr, n.value, C.byref(n))
    return list(arr)[:n.value]


def step_roofline(tensors, plan: ShardingPlan, dp: DeviceMesh, rank: int = -1,
                  layout: str = "greedy", gathers: int = 2, hbm_bw: float = B200_HBM_BW,
                  nvlink_bw: float = B200_NVLINK_BW):
    """(StepRoofline, rank) of one engine step; rank -1 = the slowest rank."""
    if isinstance(tensors, ModelSpec):
        tensors = model_tensors(tensors)
    arr = (C.c_uint64 * len(tensors))(*tensors)
    p = plan._c()
    who, out = C.c_int(), N.StepRoofline()
    _call(N.lib().amsp_step_roofline, arr, len(tensors), C.byref(p), dp._c(), rank,
          LAYOUTS[layout], gathers, hbm_bw, nvlink_bw, C.byref(who), C.byref(out))
    return StepRoofline._from(out), who.value


def solve_roofline(model: ModelSpec, cluster: ClusterSpec, profile: BandwidthProfile,
                   cfg: CostConfig = CostConfig(), hbm_bw: float = B200_HBM_BW,
                   nvlink_bw: float = B200_NVLINK_BW, layout: str = "greedy"):
    """[(PlanResult, StepRoofline)] fastest B200 step first (amsp_solve_roofline)."""
    m, _keep = model._c()
    cl, c = cluster._c(), cfg._c()
    best, bstep, n_all = N.PlanResult(), N.StepRoofline(), C.c_int()
    cap = 4096
    allr, alls = (N.PlanResult * cap)(), (N.StepRoofline * cap)()
    code = N.lib().amsp_solve_roofline(C.byref(m), C.byref(cl), profile._h, C.byref(c), hbm_bw,
                                       nvlink_bw, LAYOUTS[layout], C.byref(best),
                                       C.byref(bstep), allr, alls, cap, C.byref(n_all))
    if code == N.AMSP_EINFEASIBLE:
        raise NoFeasiblePlanError(code, N.lib().amsp_last_error().decode(),
                                  PlanResult._from(best))
    N.check(code)
    return [(PlanResult._from(allr[i]), StepRoofline._from(alls[i]))
            for i in range(min(n_all.value, cap))]


def simulate(model: ModelSpec, cluster: ClusterSpec, plan: ShardingPlan,
             profile: BandwidthProfile, cfg: CostConfig = CostConfig(),
             sim: SimConfig = SimConfig(), with_trace: bool = False) -> SimResult:
    """build_schedule + simulate_step + bubble_report (+ render_trace)."""
    m, _keep = model._c()
    cl, p, c = cluster._c(), plan._c(), cfg._c()
    k = model.modules_per_layer
    tabs = []

    def arr(v):
        if v is None:
            return None
        a = (C.c_double * k)(*v)
        tabs.append(a)
        return C.cast(a, C.POINTER(C.c_double))

    table = sim.fwd_times is not None
    sc = N.SimConfig(SimConfig.TIERS.index(sim.overlap_tier), int(sim.recompute),
                     sim.comm_streams, 1 if table else 0, sim.peak_flops_per_gpu,
                     sim.compute_efficiency, arr(sim.fwd_times),
                     arr(sim.bwd_grad_weight_times), arr(sim.bwd_grad_input_times),
                     sim.head_fwd_time, sim.head_bwd_time)
    st, idle, ne, need = C.c_double(), C.c_double(), C.c_int(), C.c_size_t()
    _call(N.lib().amsp_simulate, C.byref(m), C.byref(cl), C.byref(p), profile._h, C.byref(c),
          C.byref(sc), C.byref(st), C.byref(idle), C.byref(ne), None, 0,
          C.byref(need) if with_trace else None)
    trace = ""
    if with_trace:
        buf = C.create_string_buffer(need.value + 1)
        _call(N.lib().amsp_simulate, C.byref(m), C.byref(cl), C.byref(p), profile._h,
              C.byref(c), C.byref(sc), None, None, None, buf, need.value + 1, None)
        trace = buf.value.decode()
    return SimResult(st.value, idle.value, ne.value, trace)


# ---------------------------------------------------------------- models

def llama_model(hidden: int, layers: int, ffn: int, vocab: int, micro_batch_count: int = 1,
                micro_batch: int = 1, seq_len: int = 2048) -> ModelSpec:
    """LLaMA-shaped ModelSpec: 9 modules per layer (q,k,v,o,gate,up,down,
    attn_norm,mlp_norm); embedding, final norm and lm_head are the head
    remainder (no per-module collectives, reference domain.hpp:69-71)."""
    h, f, v = hidden, ffn, vocab
    mods = [h * h] * 4 + [f * h, f * h, h * f, h, h]
    total = layers * sum(mods) + 2 * v * h + h
    return ModelSpec(total, layers, 9, mods, hidden, seq_len, micro_batch, micro_batch_count,
                     vocab)


def llama_tensors(model: ModelSpec) -> list:
    """Flat forward order: embed, per-layer modules, final norm, lm_head."""
    head = model.vocab * model.hidden
    return [head] + list(model.module_params) * model.layer_count + [model.hidden, head]


MODELS = {
    "tiny": dict(hidden=384, layers=6, ffn=1024, vocab=8192),
    "llama-1b": dict(hidden=2048, layers=18, ffn=5632, vocab=32000),
    "llama-7b": dict(hidden=4096, layers=32, ffn=11008, vocab=32000),
    "llama-13b": dict(hidden=5120, layers=40, ffn=13824, vocab=32000),
}


def model(name: str, **kw) -> ModelSpec:
    return llama_model(**MODELS[name], **kw)
