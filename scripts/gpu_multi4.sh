mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_4.txt 2>&1
timeout 300 ./tools/p2p_bench > gpurun_out/p2p4.txt 2>&1; echo p2p4=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 ./tools/p2p_bench > gpurun_out/p2p2.txt 2>&1; echo p2p2=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_4.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
for v in 0 1 4; do
  timeout 600 $TR bench.py --gpus 4 --steps 10 --warmup 3 --variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench4_v$v.json 2> gpurun_out/bench4_v$v.err; echo bench_v$v=$?
done
timeout 900 $TR bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench=$?
timeout 600 $TR bench.py --gpus 4 --mesh 2x2 --plan p=1x1,g=2x2,os=2x2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench4_2x2.json 2> gpurun_out/bench4_2x2.err; echo bench2x2=$?
timeout 600 $TR bench.py --gpus 4 --plan p=1x1,g=1x1,os=2x1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench4_os2.json 2> gpurun_out/bench4_os2.err; echo benchos2=$?
