mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "overlap_scheduler or real_gemm" > gpurun_out/mb_pytest_eng.log 2>&1; echo eng=$?
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "sched" > gpurun_out/mb_pytest_mp.log 2>&1; echo mp=$?
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582"
Q="--no-e2e --no-cpu-baseline --steps 5 --compute gemm"
for bc in auto push; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR2 bench.py --gpus 2 $Q --bc $bc > gpurun_out/mb_n2_$bc.json 2> gpurun_out/mb_n2_$bc.err; echo n2$bc=$?
  timeout 900 $TR4 bench.py --gpus 4 $Q --bc $bc > gpurun_out/mb_n4_$bc.json 2> gpurun_out/mb_n4_$bc.err; echo n4$bc=$?
done
timeout 900 $TR4 bench.py --gpus 4 $Q --bc auto --optimizer-overlap 1 > gpurun_out/mb_n4_auto_o1.json 2> gpurun_out/mb_n4_auto_o1.err; echo n4o1=$?
