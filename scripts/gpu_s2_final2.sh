# 2-GPU box: default bench lines at HEAD (N=1, N=2), the reference arm, ncu of the W=2 default kernel (emulated, 1 GPU).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/fin_n1.json 2> gpurun_out/fin_n1.err; echo n1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29618 bench.py --gpus 2 > gpurun_out/fin_n2.json 2> gpurun_out/fin_n2.err; echo n2=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref1.json 2> gpurun_out/fin_ref1.err; echo ref1=$?
T="python tools/tune_fused.py --model llama-1b --world 2 --variants 7 --grids 296 --steps 1"
CUDA_VISIBLE_DEVICES=0 timeout 300 $T > gpurun_out/fin_v7_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step_tma -s 2 -c 1 -o gpurun_out/fin_ncu_v7_w2 $T > gpurun_out/fin_ncu_v7.log 2>&1; echo ncu=$?
