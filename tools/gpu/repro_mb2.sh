set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 1500 $TR --master-port 29614 bench.py --gpus 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4 --no-e2e --no-cpu-baseline --no-grad-ring > gpurun_out/repro_full.json 2> gpurun_out/repro_full.err; echo "full rc=$?"
grep -m6 "timed out\|Error" gpurun_out/repro_full.err
timeout 1500 $TR --master-port 29615 bench.py --gpus 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4 --no-e2e --no-cpu-baseline > gpurun_out/repro_ring.json 2> gpurun_out/repro_ring.err; echo "ring rc=$?"
grep -m6 "timed out\|Error" gpurun_out/repro_ring.err
true
