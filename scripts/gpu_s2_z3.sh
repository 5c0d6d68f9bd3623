# 4-GPU box: staged-reduce knob sweep for 13B ZeRO-3, then default bench lines (N=4 7B ZeRO-1, 13B ZeRO-3).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29615"
timeout 1500 $TR4 tools/tune_overlap.py --model llama-13b --plan zero3 --compute gemm --comm-ctas 148,296 --margins 0 --opt 1 --gather dma,tma --reduce dma > gpurun_out/z_z3_13b.jsonl 2> gpurun_out/z_z3_13b.err; echo z3=$?
timeout 1200 $TR4 bench.py --gpus 4 --model llama-13b --plan zero3 > gpurun_out/z_n4_13b.json 2> gpurun_out/z_n4_13b.err; echo b13=$?
timeout 1200 $TR4 bench.py --gpus 4 > gpurun_out/z_n4_7b.json 2> gpurun_out/z_n4_7b.err; echo b7=$?
