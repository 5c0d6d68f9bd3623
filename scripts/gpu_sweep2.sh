mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591"
timeout 1800 $TR tools/sweep.py --profile profiles/b200_nccl_4gpu.csv --out gpurun_out/sweep2_1b.jsonl > gpurun_out/sweep2.log 2>&1; echo sweep=$?
