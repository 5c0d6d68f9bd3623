# 4-GPU box: ring-depth variants 9/10 (2/4 stages): parity, W=1 sweep, N=2 / N=4 pipeline lines.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "tiny_10_steps or emulated_dp_group" > gpurun_out/s_pytest.log 2>&1; echo pt=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/tune_fused.py --model llama-7b --steps 5 --variants 9,5,10 --grids 148 > gpurun_out/s_tune7b.jsonl 2>&1; echo t7=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29619"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29620"
for v in 9 10 0; do
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 --variant $v --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/s_n2_v$v.json 2> gpurun_out/s_n2_v$v.err; echo n2v$v=$?
timeout 600 $TR4 bench.py --gpus 4 --variant $v --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/s_n4_v$v.json 2> gpurun_out/s_n4_v$v.err; echo n4v$v=$?
done
