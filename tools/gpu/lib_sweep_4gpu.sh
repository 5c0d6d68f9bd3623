# 4 GPUs: the library baseline (torch fused AdamW + NCCL RS/AG) at N=1/2/4
# and the 27-combo strategy sweep at HEAD.
set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py --impl library > gpurun_out/r02_lib1.json 2>gpurun_out/r02_lib1.err; echo "lib1 rc=$?"; tail -1 gpurun_out/r02_lib1.json
timeout 600 $TR --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 --impl library > gpurun_out/r02_lib2.json 2>gpurun_out/r02_lib2.err; echo "lib2 rc=$?"; tail -1 gpurun_out/r02_lib2.json
timeout 600 $TR --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --impl library > gpurun_out/r02_lib4.json 2>gpurun_out/r02_lib4.err; echo "lib4 rc=$?"; tail -1 gpurun_out/r02_lib4.json
timeout 1800 $TR --nproc-per-node 4 --master-port 29703 tools/sweep.py --model llama-1b --profile profiles/b200_nccl_4gpu.csv > gpurun_out/r02_sweep_1b_4gpu.jsonl 2> gpurun_out/r02_sweep.err; echo "sweep rc=$?"; tail -c 1500 gpurun_out/r02_sweep_1b_4gpu.jsonl
true
