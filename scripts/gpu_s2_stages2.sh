# 4-GPU box: 5-stage rings (11 bulk drain, 12 plain) vs 4 stages (10) at W=2 / W=4.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "tiny_10_steps or emulated_dp_group" > gpurun_out/s2b_pytest.log 2>&1; echo pt=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622"
for v in 10 11 12 8 10; do
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 --variant $v --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/s2b_n2_v$v.json 2> gpurun_out/s2b_n2_v$v.err; echo n2v$v=$?
done
for v in 10 11 12 5; do
timeout 600 $TR4 bench.py --gpus 4 --variant $v --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/s2b_n4_v$v.json 2> gpurun_out/s2b_n4_v$v.err; echo n4v$v=$?
done
