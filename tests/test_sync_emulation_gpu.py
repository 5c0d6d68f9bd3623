"""Cross-rank synchronisation of the AMSP step on ONE GPU, with the real
barrier protocol (amsp_engine_link_local_sync).

The emulated groups of tests/test_engine_gpu.py order the ranks by running
them one after another on one stream, with the barriers compiled out. Here
every rank issues on its own CUDA stream, calls are interleaved rank by
rank, and ranks > 0 are delayed by a spin kernel before they produce their
gradients. Correct results therefore REQUIRE what the multi-GPU path relies
on: barrier_kernel's st.release.sys / ld.acquire.sys flag protocol (engine
and scheduler barrier ids, epochs growing across schedulers), the
__threadfence_system release of parameter stores into peers, and the
micro-batch accumulation's release barriers. A negative control shows the
same interleaving without barriers reads stale gradients.

All ranks live in one process and one CUDA context (no time-sliced
processes waiting on each other, B200_PROFILING.md); barrier waits are
bounded (20 s -> error flag, never a hang)."""
import os

import numpy as np
import pytest

from oracle import cpu as O
from paper_2311_00257_b200 import _native as N
from paper_2311_00257_b200 import shardplan as S
from paper_2311_00257_b200.engine import DEFAULT_SEED, Engine, link_local

pytestmark = pytest.mark.gpu
if os.environ.get("CUDA_MODULE_LOADING") != "EAGER":  # tests/conftest.py sets it
    pytestmark = [pytest.mark.gpu,
                  pytest.mark.skip(reason="needs CUDA_MODULE_LOADING=EAGER (lazy loading can "
                                          "deadlock kernels that wait on each other)")]
M = S.DeviceMesh
H = O.hyper()
DELAY_NS = 3_000_000  # 3 ms: far longer than any tiny-model kernel


def _check_rank(e, want, what="rank"):
    segs, owned = e.segments()
    got = {n: e.read(n) for n in ("master", "exp_avg", "exp_avg_sq")}
    for n, ref in zip(("master", "exp_avg", "exp_avg_sq"), want[:3]):
        for f, o, ln in segs:
            assert np.array_equal(got[n][o:o + ln].view(np.uint32),
                                  ref[f:f + ln].view(np.uint32)), (what, n, f)
    if e.plan.sp() == 1:
        assert np.array_equal(e.read("params"), want[3]), (what, "params")


def _delay(stream, ns=DELAY_NS):
    N.check(N.lib().amsp_k_spin(4, ns, stream.cuda_stream))


def _streams(cuda, n):
    return [cuda.cuda.Stream() for _ in range(n)]


@pytest.mark.parametrize("world,os_k,variant", [
    (2, 2, 0), (4, 4, 0), (4, 2, 0), (8, 8, 0), (3, 3, 0),
    (2, 2, 11), (4, 4, 10), (8, 8, 6), (4, 4, 1), (2, 2, 2)])
def test_synced_group_interleaved_ranks(cuda, world, os_k, variant):
    """Rank by rank: (delay) synth grads -> step. Rank 0's step runs before
    rank 1 has even produced its gradients unless the pre-step barrier holds
    it; the post-step barrier keeps rank r from overwriting its gradients
    (next step's synth) while a peer still pulls them."""
    model = S.model("tiny")
    plan = S.ShardingPlan(M(1, 1), M(1, 1), M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r) for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    for e, s in zip(engines, streams):
        if variant:
            e.tune(variant)
        e.init_state(s)
    steps = 3
    for t in range(1, steps + 1):
        for r, (e, s) in enumerate(zip(engines, streams)):
            if r > 0:
                _delay(s)
            e.synth_grads(t, s)
            e.step(t, s)
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, steps, world, H)
    for e in engines:
        e.stats()  # raises if a barrier timed out
        _check_rank(e, want, f"rank {e.rank}")
    for e in engines:
        e.close()


def test_unsynced_interleaving_reads_stale_gradients(cuda):
    """Negative control: the same interleaving on per-rank streams with the
    barriers compiled out (link_local without sync) does NOT reproduce the
    oracle -- so the synced test above is discriminating."""
    model = S.model("tiny")
    plan = S.ShardingPlan(M(1, 1), M(1, 1), M(2, 1))
    engines = [Engine(model, plan, M(2, 1), rank=r) for r in range(2)]
    link_local(engines, sync=False)
    streams = _streams(cuda, 2)
    for e, s in zip(engines, streams):
        e.init_state(s)
    cuda.cuda.synchronize()
    for r, (e, s) in enumerate(zip(engines, streams)):
        if r > 0:
            _delay(s, 20_000_000)
        e.synth_grads(1, s)
        e.step(1, s)
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, 1, 2, H)
    with pytest.raises(AssertionError):
        _check_rank(engines[0], want)
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,dp,p,g,os_,mb", [
    (2, (2, 1), (1, 1), (2, 1), (2, 1), 3),   # ZeRO-2 (g = os)
    (4, (4, 1), (4, 1), (4, 1), (4, 1), 2),   # ZeRO-3 (s_g = s_p)
    (4, (4, 1), (2, 1), (2, 1), (4, 1), 2),   # s_g = s_p = 2 < s_os
    (4, (2, 2), (1, 1), (2, 1), (2, 1), 2),   # G shard inside each virtual node
    (8, (2, 4), (1, 1), (2, 4), (2, 4), 2),   # BASELINE partial: G shard mesh 2x4
    (4, (4, 1), (1, 1), (1, 1), (4, 1), 3)])  # ZeRO-1, in place
def test_synced_micro_batches_gradient_sharding(cuda, world, dp, p, g, os_, mb):
    """M micro-batches, rank-interleaved: every micro-batch's accumulate pulls
    the G block of each peer only after the peer's gradients are complete
    (barrier), and no rank rewrites its gradient buffer (next micro-batch)
    before every holder has pulled it (release barrier)."""
    model = S.model("tiny")
    plan = S.ShardingPlan(M(*p), M(*g), M(*os_))
    engines = [Engine(model, plan, M(*dp), rank=r, micro_batches=mb) for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    for e, s in zip(engines, streams):
        e.init_state(s)
    steps = 2
    for t in range(1, steps + 1):
        for k in range(mb):
            for r, (e, s) in enumerate(zip(engines, streams)):
                if r > 0:
                    _delay(s, 1_000_000)
                e.synth_grads(t, s, mb=k)
                if k + 1 < mb:
                    e.accumulate(t, k, s)
                else:
                    e.step(t, s)
    acc = O.accum(mb, plan.sg(), O.mesh_blocks(dp, g, world))
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, steps, world, H,
                              acc)
    for e in engines:
        e.stats()
        _check_rank(e, want, f"rank {e.rank}")
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p,os_k,mb,compute", [
    (2, 1, 2, 1, "standin"), (4, 1, 4, 1, "standin"), (4, 4, 4, 1, "standin"),
    (4, 2, 4, 2, "standin"), (2, 1, 2, 2, "standin")])
def test_synced_scheduler_two_schedulers_no_host_sync(cuda, world, p, os_k, mb, compute):
    """two schedulers on the same engines, alternating steps,
    gradients written by the grad-weight events DURING the step
    (grad_source='synth'), no host synchronisation between steps, ranks on
    their own streams. The barrier epochs must keep growing across
    schedulers, the per-bucket / per-module barriers must hold the reduces
    until every rank's gradients exist, and the end-of-step barriers must
    hold the next step's gradient writes until the owners are done."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", micro_batch_count=mb)
    g = M(p, 1) if os_k == p else M(os_k, 1)
    plan = S.ShardingPlan(M(p, 1), g, M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r, micro_batches=mb, skip_gathers=True)
               for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    prof = b200_profile()
    cost = S.CostConfig(bucket_size=1 << 20)
    sim = S.SimConfig(overlap_tier="ag_rs_ar_bc", peak_flops_per_gpu=1e18)
    scheds = [[Scheduler(e, model, prof, cost, sim, compute=compute, grad_source="synth")
               for e in engines] for k in range(2)]
    for e, s in zip(engines, streams):
        e.init_state(s)
    steps = 4
    for t in range(1, steps + 1):
        for r, s in enumerate(streams):
            if r > 0:
                _delay(s, 1_000_000)
            scheds[t % 2][r].step(t, s)
    for r, s in enumerate(streams):  # mirrored broadcast: the last step's shards
        scheds[steps % 2][r].flush(s)
    acc = O.accum(mb, plan.sg(), O.mesh_blocks((world, 1), (g.per_node, g.nodes), world))
    want = O.trajectory_range(0, engines[0].info.total_params, DEFAULT_SEED, steps, world, H,
                              acc)
    for e in engines:
        e.stats()
        _check_rank(e, want, f"rank {e.rank}")
    for k in range(2):
        for sc in scheds[k]:
            sc.close()
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p", [(2, 1), (2, 2)])
def test_synced_scheduler_real_gemm(cuda, world, p):
    """compute='gemm' on per-rank streams with real barriers: cuBLAS wgrad
    writes the gradient buffers while peers reduce finished buckets; the
    replicated parameters must come out identical on every rank."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", seq_len=256)
    plan = S.ShardingPlan(M(p, 1), M(p, 1), M(world, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r) for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    scheds = [Scheduler(e, model, b200_profile(), S.CostConfig(bucket_size=1 << 20),
                        S.SimConfig(peak_flops_per_gpu=1e15), compute="gemm")
              for e in engines]
    for e, s in zip(engines, streams):
        e.init_state(s)
    # compute-only warm-up per rank (no barriers): cuBLAS binds its per-stream
    # handles and workspaces before any rank spins on a peer
    for sc, s in zip(scheds, streams):
        sc.step(1, s, with_comm=False)
    cuda.cuda.synchronize()
    for t in (1, 2, 3):
        for r, (sc, s) in enumerate(zip(scheds, streams)):
            if r > 0:
                _delay(s, 1_000_000)
            sc.step(t, s)
    for sc, s in zip(scheds, streams):
        sc.flush(s)
    params = [e.read("params") for e in engines]
    for e in engines:
        e.stats()
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


# ---------------------------------------------------------------- gradient ring
# s_g > 1 with the gradient buffer cut to a ring (engine grad_ring): gradient
# memory is the G-shard accumulator (D_g = 2*Phi/s_g, cost_model.cpp:151) plus
# a transient ring the scheduler reuses once every rank has pulled a slot.
RING_CASES = [
    # world, dp, p, g, os, M
    (2, (2, 1), (1, 1), (2, 1), (2, 1), 1),   # ZeRO-2
    (2, (2, 1), (1, 1), (2, 1), (2, 1), 3),
    (4, (4, 1), (4, 1), (4, 1), (4, 1), 1),   # ZeRO-3
    (4, (4, 1), (4, 1), (4, 1), (4, 1), 2),
    (4, (4, 1), (2, 1), (2, 1), (4, 1), 2),   # s_g = s_p = 2 < s_os
    (4, (2, 2), (1, 1), (2, 1), (2, 1), 2),   # G shard inside each virtual node
    (8, (2, 4), (1, 1), (2, 4), (2, 4), 2)]   # BASELINE partial: G shard mesh 2x4


def _ring_group(cuda, world, dp, p, g, os_, mb, ring, reduce="sm", p2=None):
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", micro_batch_count=mb)
    plan = S.ShardingPlan(M(*p), M(*g), M(*os_), secondary_params=M(*p2) if p2 else None)
    engines = [Engine(model, plan, M(*dp), rank=r, micro_batches=mb, skip_gathers=True,
                      grad_ring=ring) for r in range(world)]
    link_local(engines, sync=True)
    cost = S.CostConfig(bucket_size=1 << 20)
    sim = S.SimConfig(overlap_tier="ag_rs_ar_bc", peak_flops_per_gpu=1e18)
    scheds = [Scheduler(e, model, b200_profile(), cost, sim, grad_source="synth", reduce=reduce)
              for e in engines]
    return model, plan, engines, scheds


@pytest.mark.parametrize("world,dp,p,g,os_,mb,reduce,p2", [c + ("sm", None) for c in RING_CASES] + [
    # the ring under copy-engine staged reduces, and with a ZeRO++ secondary mesh
    (4, (4, 1), (4, 1), (4, 1), (4, 1), 2, "dma", None),
    (2, (2, 1), (1, 1), (2, 1), (2, 1), 2, "dma", None),
    (4, (4, 1), (4, 1), (4, 1), (4, 1), 2, "sm", (2, 1))])
def test_gradient_ring_bit_exact(cuda, world, dp, p, g, os_, mb, reduce, p2):
    """Pass 1 learns the schedule's smallest ring (info.grad_ring_need) with a
    generous one; pass 2 runs 3 steps in exactly that ring -- maximal slot
    reuse, so every producer's wait on the previous occupant's release is
    exercised -- and must match the oracle bit for bit. Gradient memory drops
    from 2*Phi to the ring (+ the accumulator)."""
    phi = S.model("tiny").total_params
    _, _, engines, scheds = _ring_group(cuda, world, dp, p, g, os_, mb, 2 * phi, reduce, p2)
    need = scheds[0].info.grad_ring_need
    assert 0 < need < phi
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()
    model, plan, engines, scheds = _ring_group(cuda, world, dp, p, g, os_, mb, need, reduce, p2)
    full = Engine(S.model("tiny", micro_batch_count=mb), plan, M(*dp), rank=0,
                  micro_batches=mb, skip_gathers=True)
    assert engines[0].info.grad_elems == need
    assert full.info.device_bytes - engines[0].info.device_bytes >= 2 * (phi - need) - (1 << 20)
    full.close()
    # the allocation contract: the planner's model-state bytes (params/s_p +
    # G shard/s_g + OS/s_os, memory_breakdown = cost_model.cpp:140-160) plus
    # the transient ring and gather slots, nothing of size Phi beyond that
    mbd = S.memory_breakdown(model, plan)
    for e in engines:
        # + the greedy OS map's imbalance over Phi/s_os (few tensors in the tiny
        # model), in the OS shard and in an OS-indexed accumulator
        imbalance = (12 * max(0, e.info.owned - phi // plan.sos()) +
                     2 * max(0, e.info.acc_elems - phi // plan.sg()))
        extra = 2 * need + 2 * 2 * e.info.slot_elems + imbalance + (1 << 20)
        assert e.info.device_bytes <= mbd.d_modelstate + extra, (e.info.device_bytes,
                                                                 mbd.d_modelstate)
    streams = _streams(cuda, world)
    for e, s in zip(engines, streams):
        e.init_state(s)
    steps = 3
    for t in range(1, steps + 1):
        for r, s in enumerate(streams):
            if r > 0:
                _delay(s, 500_000)
            scheds[r].step(t, s)
    for r, s in enumerate(streams):
        scheds[r].flush(s)
    acc = O.accum(mb, plan.sg(), O.mesh_blocks(dp, g, world))
    want = O.trajectory_range(0, phi, DEFAULT_SEED, steps, world, H, acc)
    for e in engines:
        e.stats()
        _check_rank(e, want, f"rank {e.rank}")
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()


def test_gradient_ring_errors(cuda):
    model = S.model("tiny")
    with pytest.raises(N.InvalidConfig, match="s_g > 1"):
        Engine(model, S.ShardingPlan(M(1, 1), M(1, 1), M(2, 1)), M(2, 1), grad_ring=1 << 20)
    plan = S.ShardingPlan(M(1, 1), M(2, 1), M(2, 1))
    engines = [Engine(model, plan, M(2, 1), rank=r, grad_ring=1 << 10) for r in range(2)]
    link_local(engines, sync=True)
    with pytest.raises(N.InvalidConfig, match="full gradient buffer"):
        engines[0].synth_grads(1)
    with pytest.raises(N.InvalidConfig, match="full gradient buffer"):
        engines[0].step(1)
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    with pytest.raises(N.InvalidConfig, match="too small"):
        Scheduler(engines[0], model, b200_profile(), S.CostConfig(bucket_size=1 << 20),
                  S.SimConfig(peak_flops_per_gpu=1e18), grad_source="synth")
    with pytest.raises(N.InvalidConfig, match="grad-weight events"):
        Scheduler(engines[0], model, b200_profile(), S.CostConfig(bucket_size=1 << 20),
                  S.SimConfig(peak_flops_per_gpu=1e18))
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,g,mb,opt_overlap,bucket,ring", [
    (2, 2, 2, False, 1 << 20, False), (2, 2, 2, True, 1 << 20, False),
    (2, 2, 4, False, 1 << 20, False), (2, 1, 2, False, 1 << 20, False),
    (2, 2, 1, False, 1 << 20, False), (2, 2, 4, False, 1 << 27, False),
    (4, 4, 4, False, 1 << 27, False),
    # the gradient ring under real compute (bench.py's overlap_grad_ring)
    (2, 2, 4, False, 1 << 20, True), (4, 4, 2, True, 1 << 20, True)])
def test_synced_scheduler_real_gemm_micro_batches(cuda, world, g, mb, opt_overlap, bucket,
                                                  ring):
    """compute='gemm' with M micro-batches (grad-weight GEMMs produce every
    micro-batch's gradients; s_g = g > 1 folds the non-last ones into the G
    shard between backward passes), optimizer after the barrier or in
    backward, run like bench.py's overlap measurement: full steps, then
    compute-only steps, then compute + local optimizer steps, the phases
    separated by a device synchronisation. No barrier may time out and the
    replicated parameters must agree on every rank after the full steps."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", seq_len=256, micro_batch_count=mb)
    plan = S.ShardingPlan(M(1, 1), M(g, 1), M(world, 1))
    need = 0
    if ring:  # the schedule's smallest ring, learned from a generous one
        probe = [Engine(model, plan, M(world, 1), rank=r, micro_batches=mb,
                        grad_ring=model.total_params) for r in range(world)]
        link_local(probe, sync=True)
        ps = Scheduler(probe[0], model, b200_profile(), S.CostConfig(bucket_size=bucket),
                       S.SimConfig(peak_flops_per_gpu=1e15), compute="gemm")
        need = ps.info.grad_ring_need
        ps.close()
        for e in probe:
            e.close()
    engines = [Engine(model, plan, M(world, 1), rank=r, micro_batches=mb, grad_ring=need)
               for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    scheds = [Scheduler(e, model, b200_profile(), S.CostConfig(bucket_size=bucket),
                        S.SimConfig(peak_flops_per_gpu=1e15), compute="gemm",
                        optimizer_overlap=opt_overlap) for e in engines]
    for e, s in zip(engines, streams):
        e.init_state(s)
    for sc, s in zip(scheds, streams):
        sc.step(1, s, with_comm=False)
    cuda.cuda.synchronize()
    t = 0
    for _ in range(3):
        t += 1
        for r, (sc, s) in enumerate(zip(scheds, streams)):
            if r > 0:
                _delay(s, 500_000)
            sc.step(t, s)
    for sc, s in zip(scheds, streams):
        sc.flush(s)
    cuda.cuda.synchronize()
    for e in engines:
        e.stats()
    params = [e.read("params") for e in engines]
    for prm in params[1:]:
        assert np.array_equal(prm, params[0])
    # the bench's baselines: compute only, then compute + local optimizer
    for mode in (False, "optimizer", True):
        for _ in range(2):
            t += 1
            for sc, s in zip(scheds, streams):
                sc.step(t, s, with_comm=mode)
        cuda.cuda.synchronize()
    for e in engines:
        e.stats()
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()


# ---------------------------------------------------------------- ZeRO++ secondary shard
# plan.secondary_params (domain.hpp:90-97): the backward all-gathers read the
# secondary group's slices (overlap_sim.cpp:222-230, cost_model.cpp:41), each
# rank keeping Phi/s2 more bf16 (cost_model.cpp:148-150).
@pytest.mark.parametrize("gather", ["tma", "push"])
@pytest.mark.parametrize("world,p,sec", [(4, 4, 2), (8, 8, 2), (8, 8, 4), (4, 2, 2)])
def test_zeropp_secondary_shard(cuda, world, p, sec, gather):
    model = S.model("tiny")
    plan = S.ShardingPlan(M(p, 1), M(p, 1), M(world, 1) if p < world else M(p, 1),
                          secondary_params=M(sec, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r) for r in range(world)]
    link_local(engines, sync=True)
    phi = model.total_params
    plain = Engine(model, S.ShardingPlan(plan.p, plan.g, plan.os), M(world, 1))
    assert engines[0].info.secondary_shards == sec
    assert engines[0].info.secondary_elems == phi // sec
    assert engines[0].info.device_bytes - plain.info.device_bytes >= 2 * phi // sec
    plain.close()
    streams = _streams(cuda, world)
    for e, s in zip(engines, streams):
        e.tune_gather(gather)
        e.init_state(s)
    steps = 3
    for t in range(1, steps + 1):
        for r, (e, s) in enumerate(zip(engines, streams)):
            if r > 0:
                _delay(s, 300_000)
            e.synth_grads(t, s)
            e.step(t, s)
    want = O.trajectory_range(0, phi, DEFAULT_SEED, steps, world, H)
    prev = O.trajectory_range(0, phi, DEFAULT_SEED, steps - 1, world, H)
    for e in engines:
        e.stats()
        _check_rank(e, want, f"rank {e.rank}")
    # the last step's backward gathers came from the secondary slices, which
    # its forward gathers had refreshed with the step's input parameters
    offsets = np.cumsum([0] + engines[0].tensor_sizes)
    for e in engines:
        for u in range(min(2, e.info.n_units)):
            first, n, elems = e.unit(u)
            lo = offsets[first]
            assert np.array_equal(e.read(f"slot{u}", 0, elems), prev[3][lo:lo + elems]), (e.rank, u)
    # and gathering from the secondary group now reproduces them too
    e = engines[-1]
    for u in range(e.info.n_units):
        first, n, elems = e.unit(u)
        e.gather(u, u % 2, streams[-1], secondary=True)
        lo = offsets[first]
        assert np.array_equal(e.read(f"slot{u % 2}", 0, elems), prev[3][lo:lo + elems]), u
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p,sec,mb", [(4, 4, 2, 1), (4, 4, 2, 2), (8, 8, 4, 1)])
def test_zeropp_scheduler(cuda, world, p, sec, mb):
    """The overlap scheduler with a secondary mesh: each tensor's first
    all-gather of the step refreshes the secondary slice, later ones read the
    secondary group (after one barrier); the step stays bit-exact."""
    from paper_2311_00257_b200.engine import Scheduler, b200_profile
    model = S.model("tiny", micro_batch_count=mb)
    plan = S.ShardingPlan(M(p, 1), M(p, 1), M(p, 1), secondary_params=M(sec, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r, micro_batches=mb, skip_gathers=True)
               for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    scheds = [Scheduler(e, model, b200_profile(), S.CostConfig(bucket_size=1 << 20),
                        S.SimConfig(overlap_tier="ag_rs_ar_bc", peak_flops_per_gpu=1e18),
                        grad_source="synth", gather="tma") for e in engines]
    assert scheds[0].info.n_gather > 0
    for e, s in zip(engines, streams):
        e.init_state(s)
    steps = 3
    for t in range(1, steps + 1):
        for r, s in enumerate(streams):
            if r > 0:
                _delay(s, 300_000)
            scheds[r].step(t, s)
    acc = O.accum(mb, plan.sg(), O.mesh_blocks((world, 1), (p, 1), world))
    want = O.trajectory_range(0, model.total_params, DEFAULT_SEED, steps, world, H, acc)
    for e in engines:
        e.stats()
        _check_rank(e, want, f"rank {e.rank}")
    for sc in scheds:
        sc.close()
    for e in engines:
        e.close()


@pytest.mark.parametrize("world,p,os_k", [(2, 2, 2), (4, 4, 4), (4, 2, 4), (8, 8, 8)])
def test_push_all_gather_step(cuda, world, p, os_k):
    """The step's all-gather passes in push mode (every rank stores its P
    slice into its peers' slots over NVLink): bit-exact state, and after the
    last step every rank's slots hold the step's input parameters, complete
    from all peers' stores (the release fence + the barrier after the passes)."""
    model = S.model("tiny")
    plan = S.ShardingPlan(M(p, 1), M(p, 1), M(os_k, 1))
    engines = [Engine(model, plan, M(world, 1), rank=r) for r in range(world)]
    link_local(engines, sync=True)
    streams = _streams(cuda, world)
    for e, s in zip(engines, streams):
        e.tune_gather("push")
        e.init_state(s)
    steps = 3
    for t in range(1, steps + 1):
        for r, (e, s) in enumerate(zip(engines, streams)):
            if r > 0:
                _delay(s, 300_000)
            e.synth_grads(t, s)
            e.step(t, s)
    phi = model.total_params
    want = O.trajectory_range(0, phi, DEFAULT_SEED, steps, world, H)
    prev = O.trajectory_range(0, phi, DEFAULT_SEED, steps - 1, world, H)
    offsets = np.cumsum([0] + engines[0].tensor_sizes)
    for e in engines:
        e.stats()
        _check_rank(e, want, f"rank {e.rank}")
        for u in range(min(2, e.info.n_units)):
            first, n, elems = e.unit(u)
            lo = offsets[first]
            assert np.array_equal(e.read(f"slot{u}", 0, elems), prev[3][lo:lo + elems]), (e.rank, u)
    for e in engines:
        e.close()
