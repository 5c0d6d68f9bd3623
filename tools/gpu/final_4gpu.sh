# Round-end validation on 4 GPUs at HEAD: the whole GPU suite, then every
# bench line of DESIGN §6.1 (W=2 / W=4 ZeRO-1, 13B ZeRO-3 / ZeRO++, M > 1 with
# G sharding) and the reference arm.
set -x
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r02_final_pytest_4gpu.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/r02_final_pytest_4gpu.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
b() {  # name nproc args...
  local name=$1 n=$2; shift 2
  timeout 1500 $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err
  echo "$name rc=$?"; grep -m3 "Error\|timed out" gpurun_out/$name.err
}
b r02_final_n2_7b_z1 2
b r02_final_n4_7b_z1 4
b r02_final_n4_13b_z3 4 --model llama-13b --plan zero3 --no-e2e
b r02_final_n4_13b_zeropp 4 --model llama-13b --plan p=4x1,g=4x1,os=4x1,p2=2x1 --no-e2e
b r02_final_n2_7b_z2_mb4 2 --plan p=1x1,g=2x1,os=2x1 --micro-batches 4 --no-e2e
b r02_final_n4_7b_partial_mb4 4 --mesh 2x2 --plan p=1x1,g=2x2,os=2x2 --micro-batches 4 --no-e2e
timeout 900 $TR --nproc-per-node 4 --master-port 29590 bench.py --gpus 4 --impl reference > gpurun_out/r02_final_ref_n4.json 2> gpurun_out/r02_final_ref_n4.err; echo "ref rc=$?"
true
