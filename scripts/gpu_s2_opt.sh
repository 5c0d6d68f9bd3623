# 1-GPU: per-SM bandwidth of the TMA optimizer at small grids; in-backward TMA optimizer on reserved SMs.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/tune_fused.py --model llama-7b --steps 3 --variants 6,5 --grids 8,16,24,32,48,64,96,148 > gpurun_out/o_grid.jsonl 2>&1; echo grid=$?
timeout 1500 python tools/tune_overlap.py --plan replica --compute gemm --comm-ctas 16,24,32,48 --margins cc --opt 1 --opt-variant 6,5 > gpurun_out/o_ov_w1.jsonl 2>&1; echo ov=$?
timeout 600 python tools/tune_overlap.py --plan replica --compute gemm --comm-ctas 128 --margins 0 --opt 0,1 --opt-variant 0 > gpurun_out/o_ov_w1_base.jsonl 2>&1; echo base=$?
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "overlap_scheduler" > gpurun_out/o_pytest_sched.log 2>&1; echo sched=$?
