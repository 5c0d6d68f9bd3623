# Full single-GPU check at HEAD: pytest -m gpu, smoke, default bench line,
# then ncu captures of the default kernels (tools/gpu/ncu_heads.sh).
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r02_pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/r02_pytest_gpu_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/r02_bench_n1.json; tail -5 gpurun_out/r02_bench_n1.err
bash tools/gpu/ncu_heads.sh
