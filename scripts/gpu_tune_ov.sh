mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR tools/tune_overlap.py --plan zero1 > gpurun_out/tov_7b_z1.jsonl 2> gpurun_out/tov_7b_z1.err; echo a=$?
timeout 900 $TR tools/tune_overlap.py --model llama-13b --plan zero3 --comm-ctas 32,64,128 --margins 0,32 > gpurun_out/tov_13b_z3.jsonl 2> gpurun_out/tov_13b_z3.err; echo b=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/tune_overlap.py --plan replica --comm-ctas 16,32,64,128 --margins 0,16,32 > gpurun_out/tov_7b_w1.jsonl 2> gpurun_out/tov_7b_w1.err; echo c=$?
