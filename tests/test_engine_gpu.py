"""GPU parity of the AMSP step (sm_100a kernels through the C-ABI) against
the CPU oracle. The step's arithmetic is defined in oracle/amsp_oracle.c and
evaluated with explicitly rounded binary32 ops on both sides, so the bar is
BIT-EXACT for fp32 master / exp_avg / exp_avg_sq and the bf16 parameters
(stricter than north_star's 1e-5 relative / 1 ulp, which is also asserted
for documentation)."""
import numpy as np
import pytest

from oracle import cpu as O
from paper_2311_00257_b200 import shardplan as S
from paper_2311_00257_b200.engine import DEFAULT_SEED, Engine, link_local

pytestmark = pytest.mark.gpu
M = S.DeviceMesh
H = O.hyper()


def _plan(os_mesh, g_mesh=None):
    return S.ShardingPlan(M(1, 1), g_mesh or M(1, 1), os_mesh)


def _expected_from_segments(segs, owned, want):
    """Gather the oracle's per-flat-index arrays into OS-shard order."""
    out = [np.empty(owned, a.dtype) for a in want[:3]]
    for f, o, ln in segs:
        for k in range(3):
            out[k][o:o + ln] = want[k][f:f + ln]
    return out


def _expected_params(e, want_bf16):
    """The rank's parameter buffer (its P shard; everything when s_p = 1)."""
    from paper_2311_00257_b200.engine import pshard_layout
    segs, n = pshard_layout(e.tensor_sizes, e.plan.sp(), e.info.p_position, 1, 0, "contiguous")
    out = np.empty(n, np.uint16)
    for f, _, d, ln in segs:
        out[d:d + ln] = want_bf16[f:f + ln]
    return out


def _check_rank(e, want_full, steps):
    segs, owned = e.segments()
    exp = _expected_from_segments(segs, owned, want_full)
    for name, ref in zip(("master", "exp_avg", "exp_avg_sq"), exp):
        got = e.read(name)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (
            name, int(np.sum(got != ref)))
        # the north-star tolerance, stated explicitly
        np.testing.assert_allclose(got, ref, rtol=1e-5, atol=0)
    params = e.read("params")
    want = _expected_params(e, want_full[3])
    assert np.array_equal(params, want), int(np.sum(params != want))


@pytest.mark.parametrize("layout,variant", [("greedy", 0), ("contiguous", 0), ("greedy", 5),
                                            ("greedy", 1), ("greedy", 2), ("greedy", 3),
                                            ("greedy", 6), ("greedy", 7), ("greedy", 8),
                                            ("greedy", 9), ("greedy", 10), ("greedy", 11),
                                            ("greedy", 12)])
def test_single_gpu_tiny_10_steps_bit_exact(cuda, layout, variant):
    """variants 5 / 6 = the TMA bulk-copy pipeline (cp.async.bulk + mbarrier);
    7 / 8 = the same with bulk-store drains (no thread-issued global stores)."""
    model = S.model("tiny")
    e = Engine(model, _plan(M(1, 1)), M(1, 1), layout=layout)
    if variant:
        e.tune(variant)
    e.init_state()
    steps = 10
    for t in range(1, steps + 1):
        e.synth_grads(t)
        e.step(t)
    phi = e.info.total_params
    want = O.trajectory_range(0, phi, DEFAULT_SEED, steps, 1, H)
    _check_rank(e, want, steps)
    assert e.launch_count() >= 2 + 2 * steps
    e.close()


def test_ragged_tensors_scalar_path(cuda):
    # sizes that are not multiples of 8 force the element-wise tail path and
    # misaligned optimizer-state offsets
    tensors = [1003, 17, 4096, 5, 77777, 3, 8, 12345]
    for world, os_k in [(1, 1), (2, 2), (3, 3)]:
        engines = [Engine(tensors, _plan(M(os_k, 1)), M(world, 1), rank=r)
                   for r in range(world)]
        if world > 1:
            link_local(engines)
        for e in engines:
            e.init_state()
        for t in (1, 2, 3):
            for e in engines:
                e.synth_grads(t)
            for e in engines:
                e.step(t)
        want = O.trajectory_range(0, sum(tensors), DEFAULT_SEED, 3, world, H)
        for e in engines:
            _check_rank(e, want, 3)
        for e in engines:
            e.close()


@pytest.mark.parametrize("world,os_k,layout,variant", [
    (2, 2, "greedy", 0), (4, 4, "greedy", 0), (4, 2, "greedy", 0), (8, 8, "greedy", 0),
    (4, 4, "contiguous", 0), (8, 2, "contiguous", 0),
    (2, 2, "greedy", 5), (4, 4, "greedy", 6), (4, 2, "greedy", 6), (8, 8, "greedy", 6),
    (2, 2, "greedy", 7), (4, 4, "greedy", 7), (4, 2, "greedy", 8), (8, 8, "greedy", 8),
    (8, 2, "greedy", 7), (5, 5, "greedy", 8), (2, 2, "greedy", 9), (4, 4, "greedy", 10),
    (2, 2, "greedy", 11), (4, 2, "greedy", 11), (2, 2, "greedy", 12), (8, 8, "greedy", 12),
    (2, 2, "greedy", 2), (4, 4, "greedy", 1), (8, 8, "greedy", 2), (8, 2, "greedy", 1),
    # non-power-of-two groups (tensor counts not divisible by k, ragged shards)
    (3, 3, "greedy", 0), (6, 3, "greedy", 0), (6, 6, "contiguous", 0), (5, 5, "greedy", 6)])
def test_emulated_dp_group_bit_exact(cuda, world, os_k, layout, variant):
    """W ranks of one DP group emulated on one GPU (link_local): fixed-order
    fp32 gradient sum over all W ranks, AdamW on each OS shard, bf16 params
    gathered into every rank of the OS group (and replicas). Auto (0) and 5 /
    6: the TMA pipeline with W gradient sources per stage; 1 / 2: LDG."""
    model = S.model("tiny")
    plan = _plan(M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r, layout=layout) for r in range(world)]
    link_local(engines)
    for e in engines:
        if variant:
            e.tune(variant)
        e.init_state()
    steps = 4
    for t in range(1, steps + 1):
        for e in engines:
            e.synth_grads(t)
        for e in engines:
            e.step(t)
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, steps, world, H)
    owned = 0
    for e in engines:
        _check_rank(e, want, steps)
        owned += e.info.owned
    assert owned == engines[0].info.total_params * (world // os_k)
    for e in engines:
        e.close()


def test_host_buffer_step_matches_device_path(cuda):
    import torch
    model = S.model("tiny")
    e = Engine(model, _plan(M(1, 1)), M(1, 1))
    e.init_state()
    phi = e.info.total_params
    host = torch.empty(phi, dtype=torch.int16, pin_memory=True)
    for t in (1, 2):
        host.numpy().view(np.uint16)[:] = O.grads(0, phi, DEFAULT_SEED, t, 0)
        stats = e.step_host(t, host.data_ptr())
        g = (O.grads(0, phi, DEFAULT_SEED, t, 0).astype(np.uint32) << 16).view(np.float32)
        assert stats[0] == pytest.approx(float(np.sum(g.astype(np.float64) ** 2)), rel=1e-3)
    want = O.trajectory_range(0, phi, DEFAULT_SEED, 2, 1, H)
    _check_rank(e, want, 2)
    e.close()


def test_host_step_pipelined_across_chunks(cuda):
    """Single-rank host-buffer step uploads in 256M-element chunks on a copy
    stream and updates each chunk behind it: check elements on both sides of
    the chunk boundary and at the ragged tail."""
    import torch
    tensors = [200_000_000, 100_000_008, 64]
    phi = sum(tensors)
    e = Engine(tensors, _plan(M(1, 1)), M(1, 1))
    e.init_state()
    host = torch.empty(phi, dtype=torch.int16, pin_memory=True)
    for t in (1, 2):
        host.numpy().view(np.uint16)[:] = O.grads(0, phi, DEFAULT_SEED, t, 0)
        e.step_host(t, host.data_ptr())
    b = 1 << 28
    idx = np.unique(np.concatenate([np.arange(0, phi, 104729), np.arange(b - 40, b + 40),
                                    np.arange(phi - 80, phi)])).astype(np.uint64)
    want = O.trajectory(idx, DEFAULT_SEED, 2, 1, H)
    assert np.array_equal(e.read("master")[idx], want[0])
    assert np.array_equal(e.read("exp_avg_sq")[idx], want[2])
    assert np.array_equal(e.read("params")[idx], want[3])
    e.close()


def test_llama1b_sampled_after_3_steps(cuda):
    """Full-size layout (1B params, 8-way greedy OS shards emulated would need
    8x the memory; use the single-rank replica) checked on a strided sample
    plus every tensor boundary."""
    model = S.model("llama-1b")
    e = Engine(model, _plan(M(1, 1)), M(1, 1))
    e.init_state()
    for t in (1, 2, 3):
        e.synth_grads(t)
        e.step(t)
    phi = e.info.total_params
    bounds = np.cumsum([0] + S.llama_tensors(model))
    idx = np.unique(np.concatenate([np.arange(0, phi, 9973), bounds[:-1], bounds[1:] - 1,
                                    np.arange(phi - 64, phi)])).astype(np.uint64)
    want = O.trajectory(idx, DEFAULT_SEED, 3, 1, H)
    master = e.read("master")
    assert np.array_equal(master[idx], want[0])
    assert np.array_equal(e.read("exp_avg")[idx], want[1])
    assert np.array_equal(e.read("exp_avg_sq")[idx], want[2])
    assert np.array_equal(e.read("params")[idx], want[3])
    e.close()


def test_llama7b_every_element_after_2_steps(cuda):
    """The bench's default workload at full size (LLaMA-7B replica, 108 GB of
    state on one B200): every master/m/v/bf16 element bit-exact vs the oracle,
    streamed in chunks (tests/fullcheck.py)."""
    from fullcheck import check_engine
    e = Engine(S.model("llama-7b"), _plan(M(1, 1)), M(1, 1))
    e.init_state()
    for t in (1, 2):
        e.synth_grads(t)
        e.step(t)
    O.use_all_threads()
    bad = check_engine(e, 2, 1)
    e.close()
    assert not bad, bad


def test_invalid_plans_fail_loudly(cuda):
    from paper_2311_00257_b200 import _native as N
    model = S.model("tiny")
    with pytest.raises(N.InvalidConfig, match="s_g in"):
        Engine(model, S.ShardingPlan(M(1, 1), M(2, 1), M(4, 1)), M(4, 1))
    with pytest.raises(N.InvalidConfig, match="not divisible"):
        Engine([10, 7], S.ShardingPlan(M(2, 1), M(2, 1), M(2, 1)), M(2, 1))
    e = Engine(model, _plan(M(2, 1)), M(2, 1))
    with pytest.raises(N.InvalidConfig, match="peers not imported"):
        e.step(1)
    e.close()


@pytest.mark.parametrize("world,p,os_k,tier", [(1, 1, 1, "ag_rs_ar_bc"), (2, 1, 2, "ag_rs_ar_bc"),
                                               (4, 1, 4, "none"), (4, 1, 2, "ag_rs_ar"),
                                               (2, 2, 2, "ag_rs_ar_bc"), (4, 4, 4, "ag_rs"),
                                               (4, 2, 4, "ag_rs_ar_bc")])
@pytest.mark.parametrize("opt_overlap,gather,bc,ov", [(True, "sm", "auto", 0),
                                                      (False, "sm", "auto", 0),
                                                      (True, "tma", "auto", 0),
                                                      (False, "sm", "push", 0),
                                                      # in-backward optimizer on the TMA kernel
                                                      (True, "tma", "auto", 6),
                                                      (True, "sm", "push", 5),
                                                      # copy-engine staged reduces
                                                      (True, "tma", "auto", -1),
                                                      (False, "sm", "auto", -1)])
def test_overlap_scheduler_bit_exact(cuda, world, p, os_k, tier, opt_overlap, gather, bc, ov):
    """The overlap scheduler replays the reference event graph (gradient
    buckets / module reduce-scatters / all-gathers on comm streams, compute
    stand-ins on the compute stream) and its split reduce -> AdamW + push
    path gives the same bits as the oracle."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny")
    plan = S.ShardingPlan(M(p, 1), M(p, 1) if os_k == p else M(os_k, 1), M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r, skip_gathers=True) for r in range(world)]
    if world > 1:
        link_local(engines)
    prof = b200_profile()
    cost = S.CostConfig(bucket_size=1 << 20)  # several buckets on the tiny model
    sim = S.SimConfig(overlap_tier=tier, peak_flops_per_gpu=1e18)
    scheds = [Scheduler(e, model, prof, cost, sim, optimizer_overlap=opt_overlap, gather=gather,
                        bc=bc, optimizer_variant=max(ov, 0), comm_ctas=24 if ov > 0 else 0,
                        reduce="dma" if ov < 0 else "sm")
              for e in engines]
    info = scheds[0].info
    # mirrored broadcast: the graph leads with BC events (tier 4, s_p = 1, k > 1)
    assert info.mirrored_bc == int(bc == "auto" and tier == "ag_rs_ar_bc" and p == 1 and os_k > 1)
    assert info.n_events > 0 and info.n_compute > 0
    if world // p > 1 and p == 1:
        assert info.n_buckets == -(-2 * model.total_params // (1 << 20))
    if p > 1:
        assert info.n_gather > 0 and info.n_reduce == model.layer_count * model.modules_per_layer
    for e in engines:
        e.init_state()
    steps = 3
    for t in range(1, steps + 1):
        for e in engines:
            e.synth_grads(t)
        for sc in scheds:
            sc.step(t)
    for sc in scheds:  # mirrored broadcast: pull the last step's shards
        sc.flush()
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, steps, world, H)
    for e in engines:
        _check_rank(e, want, steps)
    # measured trace: same TEF schema / event names as the simulator's
    import json
    scheds[0].enable_trace(True)
    for e in engines:
        e.synth_grads(steps + 1)
    for sc in scheds:
        sc.step(steps + 1)
    measured, span_ms = scheds[0].trace()
    predicted = json.loads(scheds[0].predicted_trace())
    measured = json.loads(measured)
    assert len(measured) == len(predicted) == info.n_events
    assert sorted(x["name"] for x in measured) == sorted(x["name"] for x in predicted)
    assert span_ms > 0
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p,os_k,tier,opt_overlap,compute", [
    (2, 2, 2, "ag_rs_ar_bc", True, "standin"), (4, 4, 4, "ag_rs", False, "standin"),
    (4, 2, 4, "ag_rs_ar_bc", True, "standin"), (2, 1, 2, "ag_rs_ar_bc", False, "standin")])
def test_overlap_scheduler_recompute_graph(cuda, world, p, os_k, tier, opt_overlap, compute):
    """Activation recompute (SimConfig.recompute; overlap_sim.cpp:390-416):
    the graph re-gathers each layer before its RecomputeFwd and keeps it for
    the backward. The scheduler replays that graph (recompute events run as
    compute, the extra all-gathers as NVLink gathers) and the step stays
    bit-exact with the oracle."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", seq_len=256)
    plan = S.ShardingPlan(M(p, 1), M(p, 1) if os_k == p else M(os_k, 1), M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r, skip_gathers=True) for r in range(world)]
    if world > 1:
        link_local(engines)
    sim = S.SimConfig(overlap_tier=tier, recompute=True, peak_flops_per_gpu=1e18)
    plain = S.SimConfig(overlap_tier=tier, recompute=False, peak_flops_per_gpu=1e18)
    cost = S.CostConfig(bucket_size=1 << 20)
    scheds = [Scheduler(e, model, b200_profile(), cost, sim, optimizer_overlap=opt_overlap,
                        compute=compute) for e in engines]
    ref = Scheduler(engines[0], model, b200_profile(), cost, plain,
                    optimizer_overlap=opt_overlap)
    assert scheds[0].info.n_compute > ref.info.n_compute  # RecomputeFwd events
    if p > 1:
        assert scheds[0].info.n_gather >= ref.info.n_gather
    ref.close()
    for e in engines:
        e.init_state()
    steps = 3
    for t in range(1, steps + 1):
        for e in engines:
            e.synth_grads(t)
        for sc in scheds:
            sc.step(t)
    for sc in scheds:
        sc.flush()
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, steps, world, H)
    for e in engines:
        _check_rank(e, want, steps)
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p", [(1, 1), (2, 1), (2, 2)])
def test_scheduler_real_gemm_compute(cuda, world, p):
    """compute='gemm': linear modules run cuBLAS GEMMs of their true shapes,
    grad-weight writes the real gradient buffer the reductions read. The
    replicated / gathered parameters must stay finite and identical on every
    rank that holds them."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", seq_len=256)
    plan = S.ShardingPlan(M(p, 1), M(p, 1), M(world, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r) for r in range(world)]
    if world > 1:
        link_local(engines)
    scheds = [Scheduler(e, model, b200_profile(), S.CostConfig(bucket_size=1 << 20),
                        S.SimConfig(peak_flops_per_gpu=1e15), compute="gemm")
              for e in engines]
    for e in engines:
        e.init_state()
    for t in (1, 2):
        for sc in scheds:
            sc.step(t)
    for sc in scheds:  # mirrored broadcast (W > 1): the last step's shards
        sc.flush()
    params = [e.read("params").view(np.int16).astype(np.uint16) for e in engines]
    for prm in params:
        f = (prm.astype(np.uint32) << 16).view(np.float32)
        assert np.all(np.isfinite(f))
    if p == 1:
        for prm in params[1:]:
            assert np.array_equal(prm, params[0])
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p,os_k,layout,gather", [
    (2, 2, 2, "greedy", "sm"), (4, 4, 4, "greedy", "sm"), (4, 2, 4, "greedy", "sm"),
    (4, 2, 2, "greedy", "sm"), (4, 2, 4, "contiguous", "sm"), (8, 8, 8, "greedy", "sm"),
    (2, 2, 2, "greedy", "tma"), (4, 4, 4, "greedy", "tma"), (8, 8, 8, "greedy", "tma"),
    (4, 2, 4, "greedy", "dma"), (4, 4, 4, "greedy", "push"), (8, 8, 8, "greedy", "push")])
def test_emulated_parameter_sharding_bit_exact(cuda, world, p, os_k, layout, gather):
    """s_p > 1 (ZeRO-3 / AMSP-13B-style): intra-tensor P shards, forward and
    backward all-gathers inside the step, RS fused into the optimizer kernel;
    P shards, OS shards and gathered units checked against the oracle. The
    all-gathers run as the SM kernel, the TMA bulk-copy kernel or copy-engine
    DMAs."""
    model = S.model("tiny")
    plan = S.ShardingPlan(M(p, 1), M(p, 1) if os_k == p else M(os_k, 1), M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r, layout=layout) for r in range(world)]
    link_local(engines)
    for e in engines:
        e.tune_gather(gather)
        e.init_state()
    steps = 3
    for t in range(1, steps + 1):
        for e in engines:
            e.synth_grads(t)
        for e in engines:
            e.step(t)
    phi = engines[0].info.total_params
    want = O.trajectory_range(0, phi, DEFAULT_SEED, steps, world, H)
    for e in engines:
        assert e.info.sp == p and e.info.param_elems == phi // p
        _check_rank(e, want, steps)
    # every rank's all-gather reproduces the full updated tensors of each unit
    offsets = np.cumsum([0] + engines[0].tensor_sizes)
    e = engines[-1]
    for u in range(e.info.n_units):
        first, n, elems = e.unit(u)
        e.gather(u, u % 2)
        got = e.read(f"slot{u % 2}", 0, elems)
        lo = offsets[first]
        assert np.array_equal(got, want[3][lo:lo + elems]), (u, int(np.sum(got != want[3][lo:lo + elems])))
    for e in engines:
        e.close()


# ---------------------------------------------------------------- micro-batches
# M > 1 micro-batches per step with gradient sharding (the
# reference's T_g collectives, cost_model.cpp:119-126, overlap_sim.cpp:320-330,
# and D_g = 2*Phi/s_g, cost_model.cpp:151): bit-exact against the oracle's
# accumulation recipe (oracle/amsp_oracle.c header).
MB_CASES = [
    # world, dp, p, g, os, M
    (1, (1, 1), (1, 1), (1, 1), (1, 1), 3),   # one rank, in-place accumulation
    (2, (2, 1), (1, 1), (1, 1), (2, 1), 2),   # ZeRO-1 (s_g = 1): in place
    (4, (4, 1), (1, 1), (1, 1), (4, 1), 3),
    (2, (2, 1), (1, 1), (2, 1), (2, 1), 4),   # ZeRO-2 (g = os)
    (4, (4, 1), (1, 1), (4, 1), (4, 1), 2),
    (4, (4, 1), (1, 1), (2, 1), (2, 1), 3),   # g = os = 2: two replica blocks
    (4, (4, 1), (4, 1), (4, 1), (4, 1), 2),   # ZeRO-3 (s_g = s_p)
    (4, (4, 1), (2, 1), (2, 1), (4, 1), 3),   # s_g = s_p = 2 < s_os (AMSP-13B style)
    (8, (8, 1), (2, 1), (4, 1), (4, 1), 2),   # s_p < s_g = s_os, replicas
    (8, (2, 4), (1, 1), (2, 4), (2, 4), 2),   # BASELINE partial: G shard mesh 2x4
    (4, (2, 2), (1, 1), (2, 1), (2, 1), 2),   # 2-D mesh: G shard inside each virtual node
]


@pytest.mark.parametrize("world,dp,p,g,os_,mb", MB_CASES)
def test_micro_batches_gradient_sharding_bit_exact(cuda, world, dp, p, g, os_, mb):
    model = S.model("tiny")
    plan = S.ShardingPlan(M(*p), M(*g), M(*os_))
    engines = [Engine(model, plan, M(*dp), rank=r, micro_batches=mb) for r in range(world)]
    if world > 1:
        link_local(engines)
    for e in engines:
        e.init_state()
    steps = 3
    for t in range(1, steps + 1):
        for k in range(mb):
            for e in engines:
                e.synth_grads(t, mb=k)
            if k + 1 < mb:
                for e in engines:
                    e.accumulate(t, k)
        for e in engines:
            e.step(t)
    sg = plan.sg()
    acc = O.accum(mb, sg, O.mesh_blocks(dp, g, world))
    phi = engines[0].info.total_params
    want = O.trajectory_range(0, phi, DEFAULT_SEED, steps, world, H, acc)
    for e in engines:
        _check_rank(e, want, steps)
        # the G-shard accumulator is the plan's D_g (cost_model.cpp:151)
        info = e.info
        assert info.micro_batches == mb and info.grad_shards == sg
        if sg == 1:
            assert info.acc_elems == 0
        elif sg == plan.sp():
            assert info.acc_elems == phi // plan.sp()
            assert info.acc_sources == sg and info.acc_holders == world // sg
        else:
            assert info.acc_elems == info.owned
            assert info.acc_sources == sg and info.acc_holders == world // sg
    for e in engines:
        e.close()


def test_micro_batch_api_errors(cuda):
    model = S.model("tiny")
    e = Engine(model, _plan(M(1, 1)), M(1, 1), micro_batches=2)
    e.init_state()
    with pytest.raises(Exception, match="last micro-batch"):
        e.accumulate(1, 1)
    with pytest.raises(Exception, match="micro-batch"):
        e.synth_grads(1, mb=2)
    e.accumulate(1, 0)  # s_g = 1: in place, nothing to move
    with pytest.raises(Exception, match="micro-batches"):
        Engine(model, _plan(M(1, 1)), M(1, 1), micro_batches=17)
    e.close()
