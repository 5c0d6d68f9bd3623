mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all4_final.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo n1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR2 bench.py --gpus 2 > gpurun_out/final_n2.json 2> gpurun_out/final_n2.err; echo n2=$?
timeout 900 $TR bench.py --gpus 4 > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err; echo n4=$?
timeout 600 $TR bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/final_ref4.json 2> gpurun_out/final_ref4.err; echo ref4=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref1.json 2> gpurun_out/final_ref1.err; echo ref1=$?
