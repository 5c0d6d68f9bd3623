set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sync_emulation_gpu.py -q -p no:cacheprovider -k "gemm" > gpurun_out/r02_pytest_gemm_mb.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/r02_pytest_gemm_mb.log
bash tools/gpu/tail_ab.sh
