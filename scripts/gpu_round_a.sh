mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl library --steps 5 --warmup 2 > gpurun_out/lib1.json 2> gpurun_out/lib1.err; echo lib1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --impl library --gpus 2 --steps 5 --warmup 2 > gpurun_out/lib2.json 2> gpurun_out/lib2.err; echo lib2=$?
timeout 600 $TR bench.py --impl library --gpus 4 --steps 5 --warmup 2 > gpurun_out/lib4.json 2> gpurun_out/lib4.err; echo lib4=$?
timeout 1500 $TR tools/sweep.py --profile profiles/b200_nccl_4gpu.csv --out gpurun_out/sweep_1b.jsonl > gpurun_out/sweep.log 2>&1; echo sweep=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bdef=$?
