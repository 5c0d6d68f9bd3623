mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $TR tools/tune_gather.py > gpurun_out/tune_gather.jsonl 2> gpurun_out/tune_gather.err; echo tg=$?
timeout 900 $TR bench.py --gpus 4 --model llama-13b --plan zero3 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench4_13b_z3.json 2> gpurun_out/bench4_13b_z3.err; echo b13z3=$?
