# 4-GPU box: bulk-store drain variants 7/8 of the fused TMA kernel: parity, W=1 sweep, N=2/N=4 bench.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "tiny_10_steps or emulated_dp_group" > gpurun_out/b_pytest.log 2>&1; echo pt=$?
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "None-7 or None-8" > gpurun_out/b_pytest_multi.log 2>&1; echo ptm=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/tune_fused.py --model llama-7b --steps 5 --variants 5,7,6,8 --grids 148,296 > gpurun_out/b_tune7b.jsonl 2>&1; echo t7=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29616"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29617"
for v in 0 7 8 5; do
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 --variant $v --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/b_n2_v$v.json 2> gpurun_out/b_n2_v$v.err; echo n2v$v=$?
timeout 600 $TR4 bench.py --gpus 4 --variant $v --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/b_n4_v$v.json 2> gpurun_out/b_n4_v$v.err; echo n4v$v=$?
done
