# 4 GPUs: gradient-ring parity (one-process synced groups + torchrun groups),
# and the micro-batch / G-sharding bench lines with the ring overlap.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sync_emulation_gpu.py -q -p no:cacheprovider -k ring > gpurun_out/r02_pytest_ring_sync.log 2>&1; echo "sync ring rc=$?"; tail -15 gpurun_out/r02_pytest_ring_sync.log
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "ring or mb" > gpurun_out/r02_pytest_ring_mp.log 2>&1; echo "mp ring rc=$?"; tail -15 gpurun_out/r02_pytest_ring_mp.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
b() {  # name nproc args...
  local name=$1 n=$2; shift 2
  timeout 1500 $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err
  echo "$name rc=$?"; tail -c 300 gpurun_out/$name.json; echo; grep -m3 "Error\|error:" gpurun_out/$name.err
}
b r02_bench_n4_7b_partial_mb4 4 --mesh 2x2 --plan p=1x1,g=2x2,os=2x2 --micro-batches 4
b r02_bench_n4_7b_g2x1_mb4 4 --mesh 2x2 --plan p=1x1,g=2x1,os=2x2 --micro-batches 4
b r02_bench_n2_7b_z2_mb4 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4
