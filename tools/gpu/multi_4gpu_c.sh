# 4 GPUs: M > 1 parity with the TMA accumulator-source kernel (emulated,
# synced, torchrun), then the micro-batch / G-sharding bench lines.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_sync_emulation_gpu.py -q -p no:cacheprovider -k "micro or synced or ring or gemm" > gpurun_out/r02_pytest_mb_tma.log 2>&1; echo "emulated rc=$?"; tail -8 gpurun_out/r02_pytest_mb_tma.log
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "ring or mb" > gpurun_out/r02_pytest_mb_mp.log 2>&1; echo "mp rc=$?"; tail -5 gpurun_out/r02_pytest_mb_mp.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
b() {  # name nproc args...
  local name=$1 n=$2; shift 2
  timeout 1500 $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err
  echo "$name rc=$?"; grep -m3 "timed out\|Error" gpurun_out/$name.err
}
b r02_bench_n2_7b_z2_mb4 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4
b r02_bench_n4_7b_partial_mb4 4 --mesh 2x2 --plan p=1x1,g=2x2,os=2x2 --micro-batches 4
b r02_bench_n4_7b_g2x1_mb4 4 --mesh 2x2 --plan p=1x1,g=2x1,os=2x2 --micro-batches 4
b r02_bench_n4_13b_z3_mb2 4 --model llama-13b --plan zero3 --micro-batches 2 --no-e2e
true
