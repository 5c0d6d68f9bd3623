mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all4.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR bench.py --gpus 4 --model llama-13b --plan zero3 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench4_13b_z3.json 2> gpurun_out/bench4_13b_z3.err; echo b13z3=$?
timeout 900 $TR bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench4_7b_z1.json 2> gpurun_out/bench4_7b_z1.err; echo b7z1=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench1_7b.json 2> gpurun_out/bench1_7b.err; echo b1=$?
