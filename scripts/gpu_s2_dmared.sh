# 4-GPU box: copy-engine staged reduces in the overlap scheduler (parity + overlap sweeps).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "overlap_scheduler" > gpurun_out/d_pytest_sched.log 2>&1; echo sched=$?
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "dmared" > gpurun_out/d_pytest_multi.log 2>&1; echo multi=$?
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614"
timeout 1500 $TR4 tools/tune_overlap.py --model llama-13b --plan zero3 --compute gemm --comm-ctas 64,128 --margins 0 --opt 1 --gather dma --reduce sm,dma > gpurun_out/d_z3_13b.jsonl 2> gpurun_out/d_z3_13b.err; echo z3=$?
timeout 1200 $TR4 tools/tune_overlap.py --model llama-7b --plan zero1 --compute gemm --comm-ctas 128 --margins 0 --opt 0,1 --gather dma --reduce sm,dma > gpurun_out/d_z1_7b.jsonl 2> gpurun_out/d_z1_7b.err; echo z1=$?
