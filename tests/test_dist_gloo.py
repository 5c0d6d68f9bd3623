"""World-size-2 gloo test of the multi-rank host logic (CPU only): the IPC
handle exchange used by Engine.connect and the per-rank shard layouts /
process groups, checked for consistency across processes."""
import os
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(REPO))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2311_00257_b200 import shardplan as S
    from paper_2311_00257_b200.engine import exchange_handles, layout_segments, mesh_group
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = bytes([rank]) * 64
        got = exchange_handles(fake, world)
        assert got == [bytes([r]) * 64 for r in range(world)]
        tensors = S.llama_tensors(S.model("llama-7b"))
        res = {}
        for dp, osm in [((2, 1), (2, 1)), ((2, 1), (1, 1)), ((1, 2), (1, 2))]:
            blk, pos, mem = mesh_group(S.DeviceMesh(*dp), S.DeviceMesh(*osm), rank)
            segs, owned = layout_segments(tensors, osm[0] * osm[1], pos, "greedy")
            res[str(dp) + str(osm)] = (blk, pos, mem, segs)
        allres = [None] * world
        dist.all_gather_object(allres, res)
        q.put((rank, allres))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allres = outs[0]
    assert allres == outs[1]
    phi = sum(__import__("paper_2311_00257_b200.shardplan", fromlist=["x"]).llama_tensors(
        __import__("paper_2311_00257_b200.shardplan", fromlist=["x"]).model("llama-7b")))
    # ZeRO-1 over 2 ranks: positions 0/1, shards disjoint and covering
    k = "(2, 1)(2, 1)"
    spans = sorted((f, f + ln) for r in range(2) for f, _, ln in allres[r][k][3])
    assert spans[0][0] == 0 and spans[-1][1] == phi
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert {allres[r][k][1] for r in range(2)} == {0, 1}
    # replica OS (os=1x1): each rank owns everything, in its own block
    k = "(2, 1)(1, 1)"
    assert [allres[r][k][0] for r in range(2)] == [0, 1]
