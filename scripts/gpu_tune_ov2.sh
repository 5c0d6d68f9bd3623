mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR tools/tune_overlap.py --plan zero1 --comm-ctas 128 --margins 0 --opt 1,0 > gpurun_out/tov2_7b_z1.jsonl 2> gpurun_out/tov2_7b_z1.err; echo a=$?
timeout 900 $TR tools/tune_overlap.py --plan zero1 --compute standin --comm-ctas 128 --margins 0 --opt 1,0 > gpurun_out/tov2_7b_z1_si.jsonl 2> gpurun_out/tov2_7b_z1_si.err; echo a2=$?
timeout 900 $TR tools/tune_overlap.py --model llama-13b --plan zero3 --comm-ctas 128 --margins 0 --opt 1,0 > gpurun_out/tov2_13b_z3.jsonl 2> gpurun_out/tov2_13b_z3.err; echo b=$?
timeout 900 $TR tools/tune_overlap.py --model llama-13b --plan zero3 --compute standin --comm-ctas 128 --margins 0 --opt 1,0 > gpurun_out/tov2_13b_z3_si.jsonl 2> gpurun_out/tov2_13b_z3_si.err; echo b2=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/tune_overlap.py --plan replica --comm-ctas 128 --margins 0 --opt 1,0 > gpurun_out/tov2_7b_w1.jsonl 2> gpurun_out/tov2_7b_w1.err; echo c=$?
