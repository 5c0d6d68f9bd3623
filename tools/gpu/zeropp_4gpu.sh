# ZeRO++ secondary shard: single-process synced groups, torchrun groups, and
# the 13B bench line with the secondary mesh.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sync_emulation_gpu.py tests/test_engine_gpu.py -q -p no:cacheprovider -k "zeropp or synced or parameter_sharding or scheduler or invalid" > gpurun_out/r02_pytest_zeropp.log 2>&1; echo "sync rc=$?"; tail -25 gpurun_out/r02_pytest_zeropp.log | grep -v "^ "
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "p2 or 4x1-None-greedy-4x1" > gpurun_out/r02_pytest_zeropp_mp.log 2>&1; echo "mp rc=$?"; tail -15 gpurun_out/r02_pytest_zeropp_mp.log | grep -v "^ "
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29741 bench.py --gpus 4 --model llama-13b --plan p=4x1,g=4x1,os=4x1,p2=2x1 --no-e2e > gpurun_out/r02_bench_n4_13b_zeropp.json 2> gpurun_out/r02_bench_n4_13b_zeropp.err; echo "zeropp bench rc=$?"; grep -m3 "Error\|timed out" gpurun_out/r02_bench_n4_13b_zeropp.err
true
