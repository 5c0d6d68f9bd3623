mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_1gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
B1="python bench.py --model llama-1b --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-overlap"
timeout 300 $B1 > gpurun_out/plain_1b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step -c 1 -o gpurun_out/prof_fused_1b_v4 $B1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
B7="python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-overlap"
timeout 300 $B7 > gpurun_out/plain_7b.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b_v4.csv $B7 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$?
