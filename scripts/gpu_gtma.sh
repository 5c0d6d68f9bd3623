mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "parameter_sharding or overlap_scheduler" > gpurun_out/gt_pytest_eng.log 2>&1; echo eng=$?
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "tma" > gpurun_out/gt_pytest_mp.log 2>&1; echo mp=$?
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562"
timeout 600 $TR4 tools/tune_gather.py --model llama-13b --grids "0,-2,-1,-2,0,-2" > gpurun_out/gt_tune.jsonl 2> gpurun_out/gt_tune.err; echo tune=$?
Q="--no-e2e --no-cpu-baseline --steps 5 --plan zero3 --model llama-13b --compute gemm"
timeout 900 $TR4 bench.py --gpus 4 $Q --step-gather sm --gather dma > gpurun_out/gt_z3_sm_dma.json 2> gpurun_out/gt_z3_sm_dma.err; echo z3a=$?
timeout 900 $TR4 bench.py --gpus 4 $Q --step-gather tma --gather tma > gpurun_out/gt_z3_tma_tma.json 2> gpurun_out/gt_z3_tma_tma.err; echo z3b=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563"
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gt_pytest_mp_all.log 2>&1; echo mpall=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR2 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/gt_n2.json 2> gpurun_out/gt_n2.err; echo n2=$?
timeout 900 $TR4 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/gt_n4.json 2> gpurun_out/gt_n4.err; echo n4=$?
