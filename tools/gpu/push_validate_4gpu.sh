# The push all-gather default under real multi-process NVLink groups.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "2x1-None-greedy-2x1 or 4x1-None-greedy-4x1 or 4x1-None-greedy-2x1 or p2 or llama-13b" > gpurun_out/r02_pytest_push_mp.log 2>&1; echo "mp rc=$?"; tail -6 gpurun_out/r02_pytest_push_mp.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 $TR --nproc-per-node 4 --master-port 29811 bench.py --gpus 4 --model llama-13b --plan zero3 --no-e2e --no-grad-ring > gpurun_out/r02_final_n4_13b_z3_push.json 2> gpurun_out/r02_final_n4_13b_z3_push.err; echo "bench rc=$?"; grep -m3 "Error\|timed out" gpurun_out/r02_final_n4_13b_z3_push.err
true
