mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "single_gpu_tiny or host or llama1b" > gpurun_out/pytest_tma.log 2>&1; echo pytest=$?
timeout 600 python tools/tune_fused.py --model llama-7b --steps 5 > gpurun_out/tune_tma.jsonl 2>&1; echo tune=$?
B1="python bench.py --model llama-1b --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-overlap --variant 5"
timeout 300 $B1 > gpurun_out/plain_1b_tma.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step_tma -c 1 -o gpurun_out/prof_tma_1b $B1 > gpurun_out/ncu_tma.log 2>&1; echo ncu=$?
