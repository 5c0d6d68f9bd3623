mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sched.log 2>&1; echo pytest=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
for oo in 1 0; do
timeout 900 $TR bench.py --gpus 4 --steps 5 --warmup 2 --overlap --optimizer-overlap $oo --no-e2e --no-cpu-baseline > gpurun_out/ov4_7b_z1_o$oo.json 2> gpurun_out/ov4_7b_z1_o$oo.err; echo ov7z1_$oo=$?
timeout 900 $TR bench.py --gpus 4 --model llama-13b --plan zero3 --steps 3 --warmup 2 --overlap --optimizer-overlap $oo --no-e2e --no-cpu-baseline > gpurun_out/ov4_13b_z3_o$oo.json 2> gpurun_out/ov4_13b_z3_o$oo.err; echo ov13z3_$oo=$?
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 5 --warmup 2 --overlap --no-e2e --no-cpu-baseline > gpurun_out/ov1_7b.json 2> gpurun_out/ov1_7b.err; echo ov1=$?
