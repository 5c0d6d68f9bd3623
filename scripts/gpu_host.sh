mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/hs_pytest_mp.log 2>&1; echo mp=$?
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q > gpurun_out/hs_pytest_eng.log 2>&1; echo eng=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR2 bench.py --gpus 2 > gpurun_out/hs_n2.json 2> gpurun_out/hs_n2.err; echo n2=$?
timeout 900 $TR4 bench.py --gpus 4 > gpurun_out/hs_n4.json 2> gpurun_out/hs_n4.err; echo n4=$?
