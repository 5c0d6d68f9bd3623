# A/B of the step's all-gather passes: TMA pulls vs TMA pushes (13B ZeRO-3).
set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for g in tma push; do
  timeout 900 $TR --nproc-per-node 4 --master-port $((29800 + RANDOM % 100)) bench.py --gpus 4 --model llama-13b --plan zero3 --step-gather $g --no-overlap --no-e2e --no-cpu-baseline --no-grad-ring > gpurun_out/r02_gather_${g}_n4.json 2> gpurun_out/r02_gather_${g}_n4.err
  echo "$g n4 rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/r02_gather_${g}_n4.json').read().splitlines()[-1]); r=d['roofline']; print(d['ms_per_step'], r['step_breakdown_ms'], r.get('frac_of_phase_bound'))"
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port $((29900 + RANDOM % 100)) bench.py --gpus 2 --model llama-13b --plan zero3 --step-gather $g --no-overlap --no-e2e --no-cpu-baseline --no-grad-ring > gpurun_out/r02_gather_${g}_n2.json 2> gpurun_out/r02_gather_${g}_n2.err
  echo "$g n2 rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/r02_gather_${g}_n2.json').read().splitlines()[-1]); r=d['roofline']; print(d['ms_per_step'], r['step_breakdown_ms'], r.get('frac_of_phase_bound'))"
done
