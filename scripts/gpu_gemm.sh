mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gemm.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR bench.py --gpus 4 --steps 5 --warmup 2 --compute gemm --no-e2e --no-cpu-baseline --trace-dir gpurun_out/traces > gpurun_out/g4_7b_z1.json 2> gpurun_out/g4_7b_z1.err; echo g7z1=$?
timeout 900 $TR bench.py --gpus 4 --model llama-13b --plan zero3 --steps 3 --warmup 2 --compute gemm --no-e2e --no-cpu-baseline --trace-dir gpurun_out/traces > gpurun_out/g4_13b_z3.json 2> gpurun_out/g4_13b_z3.err; echo g13z3=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 5 --warmup 2 --compute gemm --no-e2e --no-cpu-baseline > gpurun_out/g1_7b.json 2> gpurun_out/g1_7b.err; echo g1=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --trace-dir gpurun_out/traces > gpurun_out/s1_7b.json 2> gpurun_out/s1_7b.err; echo s1=$?
