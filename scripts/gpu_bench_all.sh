mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo n1=$?
timeout 900 $TR bench.py --gpus 4 > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err; echo n4=$?
timeout 900 $TR bench.py --gpus 4 --model llama-13b --plan zero3 --no-e2e > gpurun_out/final_n4_13b.json 2> gpurun_out/final_n4_13b.err; echo n4_13=$?
timeout 600 $TR bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/final_ref4.json 2> gpurun_out/final_ref4.err; echo ref4=$?
