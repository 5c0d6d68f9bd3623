# Round-end validation on 1 GPU at HEAD (what the driver runs): the GPU suite,
# smoke, the default bench line, raw-kernel bandwidth.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r02_final_pytest_1gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r02_final_pytest_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02_final_smoke.log
timeout 900 python bench.py > gpurun_out/r02_final_n1.json 2> gpurun_out/r02_final_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_final_ref_n1.json 2> gpurun_out/r02_final_ref_n1.err; echo "ref rc=$?"
timeout 300 python tools/bench_raw.py > gpurun_out/r02_final_bench_raw.jsonl 2>&1; cat gpurun_out/r02_final_bench_raw.jsonl
