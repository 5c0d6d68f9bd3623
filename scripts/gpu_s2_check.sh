# Session-2 re-validation of HEAD on a 2-GPU box: GPU tests, smoke, N=1 and N=2 bench lines.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/s2_gpus.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/s2_n1.json 2> gpurun_out/s2_n1.err; echo n1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/s2_n2.json 2> gpurun_out/s2_n2.err; echo n2=$?
