# Push all-gather grid A/B (CTAs per SM) on 13B ZeRO-3 W=4, pipeline only.
set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in 4 2 5; do
  AMSP_PUSH_CTAS=$c timeout 600 $TR --nproc-per-node 4 --master-port $((29830 + c)) bench.py --gpus 4 --model llama-13b --plan zero3 --no-overlap --no-e2e --no-cpu-baseline --no-grad-ring > gpurun_out/r02_push_ctas$c.json 2> gpurun_out/r02_push_ctas$c.err
  python -c "import json; d=json.loads(open('gpurun_out/r02_push_ctas$c.json').read().splitlines()[-1]); r=d['roofline']; print($c, d['ms_per_step'], r['step_breakdown_ms'])"
done
