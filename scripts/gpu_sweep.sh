mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $TR tools/profile_nvlink.py --out gpurun_out/b200_nccl_4.csv > gpurun_out/profile.log 2>&1; echo prof=$?
timeout 1500 $TR tools/sweep.py --profile gpurun_out/b200_nccl_4.csv --out gpurun_out/sweep_1b.jsonl > gpurun_out/sweep.log 2>&1; echo sweep=$?
