# 4-GPU box: new auto kernels (W=2: 11, W=4: 10): multi-GPU parity, 7B full-size at W=2/4, default bench lines N=2 / N=4.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_multigpu.py -q -k "not 13b and not 2x2-2x2" > gpurun_out/f4b_multi.log 2>&1; echo multi=$?
timeout 900 python -m pytest tests/test_engine_gpu.py -q -k "emulated or host" > gpurun_out/f4b_emul.log 2>&1; echo emul=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29623 bench.py --gpus 2 > gpurun_out/f4b_n2.json 2> gpurun_out/f4b_n2.err; echo n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29624 bench.py --gpus 4 > gpurun_out/f4b_n4.json 2> gpurun_out/f4b_n4.err; echo n4=$?
