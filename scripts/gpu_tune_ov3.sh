mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR tools/tune_overlap.py --model llama-13b --plan zero3 --comm-ctas 64,128 --margins 0 --opt 1,0 --gather dma,sm > gpurun_out/tov3_13b_z3.jsonl 2> gpurun_out/tov3_13b_z3.err; echo b=$?
timeout 900 $TR tools/tune_overlap.py --model llama-13b --plan zero3 --compute standin --comm-ctas 128 --margins 0 --opt 1,0 --gather dma > gpurun_out/tov3_13b_z3_si.jsonl 2> gpurun_out/tov3_13b_z3_si.err; echo b2=$?
timeout 900 $TR tools/tune_overlap.py --model llama-13b --plan zero3 --compute gemm --seq-len 8192 --comm-ctas 128 --margins 0 --opt 0 --gather dma,sm > gpurun_out/tov3_13b_z3_8k.jsonl 2> gpurun_out/tov3_13b_z3_8k.err; echo b3=$?
