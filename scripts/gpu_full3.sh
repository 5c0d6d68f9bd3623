mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f3_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/f3_n1.json 2> gpurun_out/f3_n1.err; echo n1=$?
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572"
timeout 900 $TR4 bench.py --gpus 4 --plan zero3 --model llama-13b --no-e2e --no-cpu-baseline > gpurun_out/f3_z3.json 2> gpurun_out/f3_z3.err; echo z3=$?
