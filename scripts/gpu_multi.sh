# usage: bash scripts/gpu_multi.sh N   (run on a gpurun --gpus N box)
N=${1:-2}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$N.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for v in 0 1 2 4; do
  timeout 600 $TR bench.py --gpus $N --steps 10 --warmup 3 --variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench${N}_v$v.json 2> gpurun_out/bench${N}_v$v.err; echo bench_v$v=$?
done
timeout 900 $TR bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench$N.json 2> gpurun_out/bench$N.err; echo bench=$?
