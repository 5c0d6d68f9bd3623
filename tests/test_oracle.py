"""Pins the CPU oracle (oracle/amsp_oracle.c) before it is trusted as the
GPU checker, and checks the engine's host-side index maps.

Floating-point parity is "unpinned" by the reference (no data plane, SPEC.md
:16), so the oracle's arithmetic is checked against an independent numpy
float32 restatement of the same definitions; the index maps (greedy
inter-tensor OS layout) ARE pinned to golden output of the compiled
reference."""
import gzip
from pathlib import Path

import numpy as np
import pytest

from oracle import cpu as O
from paper_2311_00257_b200 import shardplan as S
from paper_2311_00257_b200.engine import layout_segments, mesh_group

REPO = Path(__file__).resolve().parents[1]
SEED = 0x414D5350


def bf16_rne(x: np.ndarray) -> np.ndarray:
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def test_bf16_matches_torch_rne():
    import torch
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 20, 100000))).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bf16_rne(x), want)
    # oracle's own conversion, through the master->param path
    idx = np.arange(5000, dtype=np.uint64)
    master, _, _, param = O.trajectory(idx, SEED, 0, 1, O.hyper())
    assert np.array_equal(param, bf16_rne(master))


def numpy_trajectory(idx, steps, world, h):
    """Independent float32 restatement of the oracle definitions."""
    f32 = np.float32
    p = np.array([O.master_init(SEED, int(i)) for i in idx], np.float32)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for t in range(1, steps + 1):
        bc1 = 1.0 - h.beta1 ** t
        bc2 = 1.0 - h.beta2 ** t
        b1, omb1 = f32(h.beta1), f32(1.0 - h.beta1)
        b2, omb2 = f32(h.beta2), f32(1.0 - h.beta2)
        step_size = f32(h.lr / bc1)
        inv = f32(1.0 / np.sqrt(bc2))
        eps, decay, scale = f32(h.eps), f32(1.0 - h.lr * h.weight_decay), f32(1.0 / world)
        g = None
        for r in range(world):
            gr = np.array([O.lib().amsp_o_grad_bf16(SEED, t, r, int(i)) for i in idx],
                          np.uint16).astype(np.uint32) << 16
            gr = gr.view(np.float32)
            g = gr if g is None else (g + gr).astype(np.float32)
        g = (g * scale).astype(np.float32)
        m = (b1 * m + omb1 * g).astype(np.float32)
        v = (b2 * v + (omb2 * g) * g).astype(np.float32)
        d = (np.sqrt(v) * inv + eps).astype(np.float32)
        p = (p * decay).astype(np.float32)
        p = (p - step_size * (m / d)).astype(np.float32)
    return p, m, v, bf16_rne(p)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_oracle_matches_numpy_restatement(world):
    idx = np.concatenate([np.arange(0, 300), np.array([2**33 + 5, 6_738_415_615])]).astype(np.uint64)
    h = O.hyper()
    got = O.trajectory(idx, SEED, 4, world, h)
    want = numpy_trajectory(idx, 4, world, h)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_oracle_agrees_with_torch_adamw(world):
    """Independent check of the oracle's update against torch.optim.AdamW
    (single-tensor fp32 CPU path; the optimizer a PyTorch executor such as the
    paper's InternEvo would run) on the same fp32-reduced gradients. Its
    operation order differs (lerp for m, sqrt(v)/sqrt(bc2) for the
    denominator), so agreement is to the north-star tolerance (1e-5 relative
    on master, m and v after 10 steps, with small absolute floors for values
    that pass through zero), not bit-exact."""
    import torch
    n, steps = 1 << 14, 10
    start = 6_000_000_000  # inside the 7B flat index space
    h = O.hyper()
    want = O.trajectory_range(start, n, SEED, steps, world, h)
    p0 = np.array([O.master_init(SEED, start + i) for i in range(n)], np.float32)
    param = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.AdamW([param], lr=h.lr, betas=(h.beta1, h.beta2), eps=h.eps,
                            weight_decay=h.weight_decay, foreach=False, fused=False)
    for t in range(1, steps + 1):
        g = None
        for r in range(world):  # fixed rank order, fp32 sum, then 1/W (exact here)
            gr = (O.grads(start, n, SEED, t, r).astype(np.uint32) << 16).view(np.float32)
            g = gr.copy() if g is None else (g + gr).astype(np.float32)
        param.grad = torch.from_numpy((g * np.float32(1.0 / world)).astype(np.float32))
        opt.step()
    st = opt.state[param]
    np.testing.assert_allclose(param.detach().numpy(), want[0], rtol=1e-5, atol=1e-5 * h.lr)
    # moments: relative, with a floor of 1e-6 of the gradient scale (|g| <= 2^-7)
    # for moments that pass through zero
    gmax = 2.0 ** -7
    np.testing.assert_allclose(st["exp_avg"].numpy(), want[1], rtol=1e-5, atol=1e-6 * gmax)
    np.testing.assert_allclose(st["exp_avg_sq"].numpy(), want[2], rtol=1e-5,
                               atol=1e-6 * gmax * gmax)


def test_gradient_definition():
    g = O.grads(0, 100000, SEED, 3, 1).astype(np.uint32) << 16
    f = g.view(np.float32)
    assert np.all(np.abs(f) <= 2.0 ** -7)
    assert abs(f.mean()) < 1e-4 and f.std() > 1e-3
    # distinct ranks / steps give distinct streams
    assert not np.array_equal(O.grads(0, 64, SEED, 3, 0), O.grads(0, 64, SEED, 3, 1))
    assert not np.array_equal(O.grads(0, 64, SEED, 3, 0), O.grads(0, 64, SEED, 4, 0))


def _golden_greedy():
    text = gzip.decompress((REPO / "tests/golden/plan_dump.txt.gz").read_bytes()).decode()
    out = {}
    for line in text.splitlines():
        if line.startswith("greedy ") and " assign " in line and "rnd" not in line:
            head, assign = line.split(" assign ")
            parts = head.split()
            name, k = parts[1], int(parts[2][2:])
            sizes = [int(x) for x in head.split(" sizes ")[1].split()]
            out[(name, k)] = ([int(a) for a in assign.split()], sizes)
    return out


@pytest.mark.parametrize("name,model", [("tiny", "tiny"), ("1B", "llama-1b"),
                                        ("7B", "llama-7b"), ("13B", "llama-13b")])
def test_index_map_pinned_to_reference(name, model):
    gold = _golden_greedy()
    tensors = S.llama_tensors(S.model(model))
    for k in (1, 2, 3, 4, 8, 16):
        want_assign, want_sizes = gold[(name, k)]
        assert O.partition_greedy(tensors, k) == (want_assign, want_sizes)
        assert S.partition_tensors_greedy(tensors, k) == (want_assign, want_sizes)
        # the engine's per-rank segments realise exactly that assignment
        offsets = np.concatenate([[0], np.cumsum(tensors)])
        for shard in range(k):
            segs, owned = layout_segments(tensors, k, shard, "greedy")
            assert owned == want_sizes[shard]
            covered = set()
            for f, o, ln in segs:
                t0 = int(np.searchsorted(offsets, f))
                end = f + ln
                t = t0
                while offsets[t] < end:
                    assert want_assign[t] == shard
                    covered.add(t)
                    t += 1
            assert covered == {t for t, a in enumerate(want_assign) if a == shard}


@pytest.mark.parametrize("layout", ["greedy", "contiguous"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_layout_partitions_flat_vector(layout, k):
    tensors = S.llama_tensors(S.model("llama-7b"))
    phi = sum(tensors)
    spans = []
    for shard in range(k):
        segs, owned = layout_segments(tensors, k, shard, layout)
        assert sum(s[2] for s in segs) == owned
        assert [s[1] for s in segs] == list(np.cumsum([0] + [s[2] for s in segs[:-1]]))
        spans += [(f, f + ln) for f, _, ln in segs]
    spans.sort()
    assert spans[0][0] == 0 and spans[-1][1] == phi
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    if layout == "contiguous":
        assert all(f % 8 == 0 for f, _ in spans)


def test_ragged_and_degenerate_layouts():
    tensors = [3, 5, 7, 1, 9]
    for k in (1, 2, 5, 7):
        total = 0
        for shard in range(k):
            _, owned = layout_segments(tensors, k, shard, "greedy")
            total += owned
        assert total == sum(tensors)
    with pytest.raises(Exception):
        layout_segments(tensors, 2, 2, "greedy")


def test_mesh_groups():
    dp = S.DeviceMesh(2, 4)
    seen = {}
    for r in range(8):
        blk, pos, mem = mesh_group(dp, S.DeviceMesh(2, 2), r)
        assert mem[pos] == r
        seen.setdefault(blk, set()).update(mem)
    assert sorted(map(sorted, seen.values())) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    blk, pos, mem = mesh_group(S.DeviceMesh(4, 1), S.DeviceMesh(2, 1), 3)
    assert (blk, pos, mem) == (1, 1, [2, 3])


@pytest.mark.parametrize("sp,k", [(2, 1), (2, 2), (4, 2), (8, 1), (4, 4)])
@pytest.mark.parametrize("layout", ["greedy", "contiguous"])
def test_pshard_layout_partitions(sp, k, layout):
    from paper_2311_00257_b200.engine import pshard_layout
    tensors = S.llama_tensors(S.model("tiny"))
    phi = sum(tensors)
    flat_spans = []
    for p_pos in range(sp):
        dst_spans = []
        owned_total = 0
        for os_pos in range(k):
            segs, owned = pshard_layout(tensors, sp, p_pos, k, os_pos, layout)
            owned_total += owned
            assert sum(s[3] for s in segs) == owned
            flat_spans += [(f, f + ln) for f, _, _, ln in segs]
            dst_spans += [(d, d + ln) for _, _, d, ln in segs]
        assert owned_total == phi // sp
        dst_spans.sort()
        assert dst_spans[0][0] == 0 and dst_spans[-1][1] == phi // sp
        assert all(a[1] == b[0] for a, b in zip(dst_spans, dst_spans[1:]))
    flat_spans.sort()
    assert flat_spans[0][0] == 0 and flat_spans[-1][1] == phi
    assert all(a[1] == b[0] for a, b in zip(flat_spans, flat_spans[1:]))
    with pytest.raises(Exception, match="not divisible"):
        pshard_layout([10, 7], 2, 0, 1, 0, layout)


def test_fullcheck_streams_every_element_and_catches_a_flip():
    """tests/fullcheck.py (the full-size GPU parity checker) on a host-side
    stand-in engine: rank 1 of a 2-rank ZeRO-1 greedy layout of the tiny model,
    buffers filled from the oracle; one flipped bit in each buffer is found."""
    from types import SimpleNamespace

    from fullcheck import check_engine
    from paper_2311_00257_b200.engine import DEFAULT_SEED, pshard_layout
    sizes = S.llama_tensors(S.model("tiny"))
    segs, owned = pshard_layout(sizes, 1, 0, 2, 1, "greedy")
    phi = sum(sizes)
    want = O.trajectory_range(0, phi, DEFAULT_SEED, 2, 2, O.hyper())
    bufs = {"params": want[3].copy()}
    for name, ref in zip(("master", "exp_avg", "exp_avg_sq"), want[:3]):
        b = np.empty(owned, np.float32)
        for f, o, _, ln in segs:
            b[o:o + ln] = ref[f:f + ln]
        bufs[name] = b

    class Fake:
        tensor_sizes = sizes
        plan = SimpleNamespace(sp=lambda: 1)
        info = SimpleNamespace(p_position=0, owned=owned)

        def segments(self):
            return [(f, o, ln) for f, o, _, ln in segs], owned

        def read(self, which, off, n):
            return bufs[which][off:off + n].copy()

    logs = []
    assert check_engine(Fake(), 2, 2, chunk=1 << 20, log=logs.append) == []
    assert f"{phi} params + {owned} x 3" in logs[0]
    for name in ("params", "master", "exp_avg_sq"):
        b = bufs[name]
        b.view(np.uint16 if name == "params" else np.uint32)[owned // 3] ^= 1
        bad = check_engine(Fake(), 2, 2, chunk=1 << 20, log=logs.append)
        assert len(bad) == 1 and bad[0].startswith(name), bad
        b.view(np.uint16 if name == "params" else np.uint32)[owned // 3] ^= 1


# ---------------------------------------------------------------- micro-batches
# Gradient accumulation over M micro-batches and gradient sharding (s_g > 1),
# PAPER.md:316-326 / cost_model.cpp:119-126: an independent numpy restatement
# of the recipe in the oracle's header (own splitmix64, own bf16 rounding).

def _splitmix64(x: np.ndarray) -> np.ndarray:
    z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
    return z ^ (z >> np.uint64(31))


def np_grad(idx, t, mb, r) -> np.ndarray:
    key = (np.uint64(SEED) ^ np.uint64(t << 48) ^ np.uint64(mb << 44) ^ np.uint64(r << 40)
           ^ idx.astype(np.uint64))
    q = (_splitmix64(key) >> np.uint64(40)).astype(np.int64) - (1 << 23)
    u = q.astype(np.float32) * np.float32(1.0 / 8388608.0)
    return bf16_rne((u * np.float32(0.0078125)).astype(np.float32))


def up(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def np_reduced(idx, t, world, M, staged, block_of):
    f32 = np.float32
    if M == 1:
        g = up(np_grad(idx, t, 0, 0))
        for r in range(1, world):
            g = (g + up(np_grad(idx, t, 0, r))).astype(f32)
        return g
    if not staged:
        g = None
        for r in range(world):
            acc = np_grad(idx, t, 0, r)
            for mb in range(1, M):
                acc = bf16_rne((up(acc) + up(np_grad(idx, t, mb, r))).astype(f32))
            g = up(acc) if g is None else (g + up(acc)).astype(f32)
        return g
    g = None
    for b in range(max(block_of) + 1):
        members = [r for r in range(world) if block_of[r] == b]
        acc = None
        for mb in range(M - 1):
            s = None
            for r in members:
                x = up(np_grad(idx, t, mb, r))
                if s is None:
                    s = x if mb == 0 else (up(acc) + x).astype(f32)
                else:
                    s = (s + x).astype(f32)
            acc = bf16_rne(s)
        g = up(acc) if g is None else (g + up(acc)).astype(f32)
    for r in range(world):
        g = (g + up(np_grad(idx, t, M - 1, r))).astype(f32)
    return g


ACCUM_CASES = [(2, 2, 0, [0, 1]), (4, 3, 0, [0, 1, 2, 3]),          # s_g = 1, in place
               (2, 2, 1, [0, 0]), (4, 4, 1, [0, 0, 0, 0]),          # ZeRO-2/3, one block
               (4, 2, 1, [0, 0, 1, 1]), (4, 3, 1, [0, 1, 0, 1]),    # replica blocks, 2-D mesh
               (8, 2, 1, O.mesh_blocks((2, 4), (2, 4), 8)), (8, 4, 1, O.mesh_blocks((8, 1), (4, 1), 8))]


@pytest.mark.parametrize("world,M,staged,block_of", ACCUM_CASES)
def test_oracle_microbatch_recipe_matches_numpy(world, M, staged, block_of):
    idx = np.concatenate([np.arange(0, 257), np.array([2**33 + 5, 13_015_864_319])]).astype(np.uint64)
    acc = O.accum(M, 2 if staged else 1, block_of)
    for t in (1, 3):
        want = np_reduced(idx, t, world, M, staged, block_of)
        got = np.array([O.reduced_grad(SEED, t, int(i), world, acc) for i in idx], np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # micro-batch 0 is the single-micro-batch gradient (same key)
    assert np.array_equal(O.grads_mb(10, 64, SEED, 2, 0, 1), O.grads(10, 64, SEED, 2, 1))
    assert np.array_equal(O.grads_mb(10, 64, SEED, 2, 3, 1),
                          np_grad(np.arange(10, 74, dtype=np.uint64), 2, 3, 1))


def test_oracle_microbatch_one_is_flat_sum():
    idx = np.arange(0, 500, dtype=np.uint64)
    h = O.hyper()
    flat = O.trajectory(idx, SEED, 3, 4, h)
    for staged, blocks in ((0, [0, 1, 2, 3]), (1, [0, 1, 0, 1])):
        got = O.trajectory(idx, SEED, 3, 4, h, O.accum(1, 2 if staged else 1, blocks))
        for a, b in zip(got, flat):
            assert np.array_equal(a, b)


def test_oracle_microbatch_scale_and_mean():
    """The step's gradient is the mean over W*M micro-batch gradients: with
    M = 4 the Adam step sees scale 1/(W*M), and the staged sum is within bf16
    accumulation error of the exact fp64 mean."""
    idx = np.arange(0, 2000, dtype=np.uint64)
    world, M = 2, 4
    acc = O.accum(M, 2, [0, 0])
    exact = sum(up(np_grad(idx, 1, mb, r)).astype(np.float64)
                for mb in range(M) for r in range(world))
    got = np.array([O.reduced_grad(SEED, 1, int(i), world, acc) for i in idx], np.float64)
    assert np.max(np.abs(got - exact)) <= 2 ** -8 * np.max(np.abs(exact)) * M
    s = O.scalars(1, world * M, O.hyper())
    assert s.grad_scale == np.float32(1.0 / 8)


def test_oracle_mesh_blocks_match_engine_groups():
    """The checker's block map equals the engine's process groups."""
    for dp, mesh in [((8, 1), (4, 1)), ((2, 4), (2, 4)), ((2, 4), (2, 2)), ((4, 2), (2, 1)),
                     ((2, 2), (1, 2)), ((4, 1), (1, 1))]:
        world = dp[0] * dp[1]
        blocks = O.mesh_blocks(dp, mesh, world)
        for r in range(world):
            blk, _, _ = mesh_group(S.DeviceMesh(*dp), S.DeviceMesh(*mesh), r)
            assert blk == blocks[r]
