mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parameter_sharding or torchrun" > gpurun_out/pytest_z3.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR bench.py --gpus 4 --model llama-13b --plan zero3 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench4_13b_z3.json 2> gpurun_out/bench4_13b_z3.err; echo b13z3=$?
timeout 900 $TR bench.py --gpus 4 --plan p=2x1,g=2x1,os=4x1 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench4_7b_p2.json 2> gpurun_out/bench4_7b_p2.err; echo b7p2=$?
