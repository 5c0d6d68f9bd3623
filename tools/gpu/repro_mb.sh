set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 900 $TR --master-port 29611 bench.py --gpus 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4 --model llama-1b --compute gemm --no-e2e --no-cpu-baseline --no-grad-ring --steps 3 > gpurun_out/repro_1b.json 2> gpurun_out/repro_1b.err; echo "1b rc=$?"
grep -m5 "timed out\|Error" gpurun_out/repro_1b.err
timeout 900 $TR --master-port 29612 bench.py --gpus 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4 --compute gemm --no-e2e --no-cpu-baseline --no-grad-ring --steps 3 > gpurun_out/repro_7b.json 2> gpurun_out/repro_7b.err; echo "7b rc=$?"
grep -m5 "timed out\|Error" gpurun_out/repro_7b.err
timeout 900 $TR --master-port 29613 bench.py --gpus 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4 --compute standin --no-e2e --no-cpu-baseline --no-grad-ring --steps 3 > gpurun_out/repro_7b_si.json 2> gpurun_out/repro_7b_si.err; echo "7b standin rc=$?"
grep -m5 "timed out\|Error" gpurun_out/repro_7b_si.err
