# ZeRO++ secondary shard: single-process synced groups and torchrun groups.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sync_emulation_gpu.py tests/test_engine_gpu.py -q -p no:cacheprovider -k "zeropp or synced or ring or parameter_sharding or invalid" > gpurun_out/r02_pytest_zeropp.log 2>&1; echo "sync rc=$?"; tail -25 gpurun_out/r02_pytest_zeropp.log | grep -v "^ "
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "p2 or 4x1-None-greedy-4x1-0" > gpurun_out/r02_pytest_zeropp_mp.log 2>&1; echo "mp rc=$?"; tail -15 gpurun_out/r02_pytest_zeropp_mp.log | grep -v "^ "
true
