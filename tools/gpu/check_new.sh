# new-kernel / sync-emulation checks on one GPU, then raw-kernel bandwidth
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sync_emulation_gpu.py tests/test_kernels_gpu.py -x -q -p no:cacheprovider > gpurun_out/r02_pytest_sync_raw.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02_pytest_sync_raw.log
timeout 300 python tools/bench_raw.py > gpurun_out/r02_bench_raw.jsonl 2> gpurun_out/r02_bench_raw.err; echo "raw rc=$?"
cat gpurun_out/r02_bench_raw.jsonl; tail -5 gpurun_out/r02_bench_raw.err
