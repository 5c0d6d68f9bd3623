mkdir -p gpurun_out
timeout 900 python tools/tune_fused.py --model llama-1b --world 8 --variants 0,5,6,2,1 --grids 0 --steps 3 > gpurun_out/w8_tune.jsonl 2>&1; echo w8=$?
timeout 900 python tools/tune_fused.py --model llama-1b --world 4 --variants 0,5,6,2 --grids 0 --steps 3 > gpurun_out/w4_tune.jsonl 2>&1; echo w4=$?
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -k "emulated_dp_group" > gpurun_out/w8_pytest.log 2>&1; echo emu=$?
