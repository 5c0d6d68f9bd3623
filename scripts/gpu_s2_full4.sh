# 4-GPU box: W=8 oversubscribed parity, full-size every-element parity, N=8 bench functional check.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k oversub > gpurun_out/f4_oversub.log 2>&1; echo oversub=$?
timeout 2400 python -m pytest tests/test_multigpu.py tests/test_engine_gpu.py -x -q -k "every_element" --durations=0 > gpurun_out/f4_fullsize.log 2>&1; echo full=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 8 --steps 3 --warmup 3 --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/f4_n8_oversub.json 2> gpurun_out/f4_n8_oversub.err; echo n8=$?
