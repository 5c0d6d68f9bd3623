set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29741 bench.py --gpus 4 --model llama-13b --plan p=4x1,g=4x1,os=4x1,p2=2x1 --no-e2e > gpurun_out/r02_bench_n4_13b_zeropp.json 2> gpurun_out/r02_bench_n4_13b_zeropp.err; echo "zeropp rc=$?"; grep -m3 "Error\|timed out" gpurun_out/r02_bench_n4_13b_zeropp.err
true
