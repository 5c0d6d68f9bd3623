mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f4_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo smoke=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/f4_n1.json 2> gpurun_out/f4_n1.err; echo n1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR2 bench.py --gpus 2 > gpurun_out/f4_n2.json 2> gpurun_out/f4_n2.err; echo n2=$?
timeout 900 $TR4 bench.py --gpus 4 > gpurun_out/f4_n4.json 2> gpurun_out/f4_n4.err; echo n4=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f4_ref1.json 2> gpurun_out/f4_ref1.err; echo ref1=$?
timeout 600 $TR4 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/f4_ref4.json 2> gpurun_out/f4_ref4.err; echo ref4=$?
