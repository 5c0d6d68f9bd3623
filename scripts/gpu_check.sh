mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python tools/tune_fused.py --model llama-7b --steps 5 > gpurun_out/tune7b.jsonl 2>&1; echo tune=$?
timeout 300 python tools/tune_fused.py --model llama-1b --world 4 --variants 0,1,2,3 --grids 0,-1 > gpurun_out/tune1b_w4.jsonl 2>&1; echo tune4=$?
B1="python bench.py --model llama-1b --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $B1 > gpurun_out/plain_1b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_step -c 1 -o gpurun_out/prof_fused_1b $B1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
B7="python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $B7 > gpurun_out/plain_7b.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b.csv $B7 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$?
