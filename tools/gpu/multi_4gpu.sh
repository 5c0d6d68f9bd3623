# 4-GPU box: the whole GPU suite (real multi-process NVLink groups), then the
# bench lines at W=2 / W=4 (7B ZeRO-1, 13B ZeRO-3, the 2x2 partial plan,
# micro-batches with G sharding) and the reference arm.
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r02_topo_4gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r02_pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02_pytest_gpu_4gpu.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
b() {  # name nproc args...
  local name=$1 n=$2; shift 2
  timeout 1200 $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err
  echo "$name rc=$?"; tail -c 600 gpurun_out/$name.json; echo
}
b r02_bench_n2_7b_z1 2
b r02_bench_n4_7b_z1 4
b r02_bench_n4_13b_z3 4 --model llama-13b --plan zero3
b r02_bench_n4_7b_partial_mb1 4 --mesh 2x2 --plan p=1x1,g=2x2,os=2x2
# M > 1 micro-batches with G sharding (+ the gradient-ring overlap line)
b r02_bench_n2_7b_z2_mb4 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4
b r02_bench_n4_7b_partial_mb4 4 --mesh 2x2 --plan p=1x1,g=2x2,os=2x2 --micro-batches 4
b r02_bench_n4_13b_z3_mb2 4 --model llama-13b --plan zero3 --micro-batches 2 --no-e2e
timeout 900 $TR --nproc-per-node 4 --master-port 29590 bench.py --gpus 4 --impl reference > gpurun_out/r02_ref_n4.json 2> gpurun_out/r02_ref_n4.err; echo "ref rc=$?"; tail -c 800 gpurun_out/r02_ref_n4.json
