"""B200 collective profiler -> the reference's profile CSV.

  torchrun --nproc-per-node N tools/profile_nvlink.py --out profiles/b200_nccl_N.csv

Measures NCCL AllGather / ReduceScatter / AllReduce / Broadcast (bf16) over
every single-node sub-mesh a x 1 (a | N, a > 1; groups are contiguous rank
blocks, as in the engine's mesh semantics) at message sizes 1 KiB .. 1 GiB
and writes `op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s` rows.
As the reference consumes it (comm_model.cpp:121-127: t = v / w, v = the
full message size named by each cost formula), the column holds ALGBW =
message bytes / time, not nccl-tests busbw. The CSV loads with
shardplan.BandwidthProfile.load / amsp_profile_load and feeds solve().
"""
import argparse
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rows = []
    sizes = [1 << k for k in range(args.min_log2, args.max_log2 + 1, 2)]
    for a in [d for d in range(2, world + 1) if world % d == 0]:
        groups = [dist.new_group(list(range(b * a, (b + 1) * a))) for b in range(world // a)]
        g = groups[rank // a]
        me = rank % a
        for v in sizes:
            n = v // 2  # bf16 elements of the full message
            n -= n % a
            full = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            shard = torch.empty(n // a, dtype=torch.bfloat16, device="cuda")
            ops = {
                "allgather": lambda: dist.all_gather_into_tensor(full, shard, group=g),
                "reducescatter": lambda: dist.reduce_scatter_tensor(shard, full, group=g),
                "allreduce": lambda: dist.all_reduce(full, group=g),
                "broadcast": lambda: dist.broadcast(full, src=(rank // a) * a, group=g),
            }
            for name, fn in ops.items():
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                dist.barrier()
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                for _ in range(args.iters):
                    fn()
                t1.record()
                torch.cuda.synchronize()
                ms = torch.tensor([t0.elapsed_time(t1) / args.iters], device="cuda")
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
                bw = (n * 2) / (float(ms) * 1e-3)
                if rank == 0:
                    rows.append(f"{name},{n * 2},{a},1,{bw:.6e}")
            del full, shard
        del me
    if rank == 0:
        text = "op,size_bytes,gpus_per_node,nodes,bus_bw_bytes_per_s\n" + "\n".join(rows) + "\n"
        if args.out:
            Path(args.out).write_text(text)
        print(text)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
