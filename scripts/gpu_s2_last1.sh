# 1-GPU box: final sanity at HEAD (single-GPU suite, smoke, default N=1 line, N=2 oversubscribed functional line).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/last_pytest1.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/last_n1.json 2> gpurun_out/last_n1.err; echo n1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29625 bench.py --gpus 2 --model llama-1b --steps 3 --warmup 3 --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/last_n2_oversub.json 2> gpurun_out/last_n2_oversub.err; echo n2o=$?
