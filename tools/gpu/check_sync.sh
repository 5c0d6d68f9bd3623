set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sync_emulation_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider --durations=15 > gpurun_out/r02_pytest_sync_raw.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r02_pytest_sync_raw.log
timeout 300 python tools/bench_raw.py > gpurun_out/r02_bench_raw.jsonl 2>&1; cat gpurun_out/r02_bench_raw.jsonl
