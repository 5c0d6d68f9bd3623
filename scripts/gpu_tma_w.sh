mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "emulated_dp_group" > gpurun_out/tw_pytest_emu.log 2>&1; echo emu=$?
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/tw_pytest_mp.log 2>&1; echo mp=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542"
Q="--no-overlap --no-e2e --no-cpu-baseline --steps 10"
for v in 0 5 6; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 $Q --variant $v > gpurun_out/tw_n2_v$v.json 2> gpurun_out/tw_n2_v$v.err; echo n2v$v=$?
  timeout 600 $TR4 bench.py --gpus 4 $Q --variant $v > gpurun_out/tw_n4_v$v.json 2> gpurun_out/tw_n4_v$v.err; echo n4v$v=$?
done
timeout 600 $TR4 bench.py --gpus 4 $Q --variant 5 --plan zero3 --model llama-13b > gpurun_out/tw_n4_z3_v5.json 2> gpurun_out/tw_n4_z3_v5.err; echo z3v5=$?
