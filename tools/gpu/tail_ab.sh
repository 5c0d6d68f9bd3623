# A/B of the overlapped step's end-of-step optimizer kernel at W=1 (LDG auto
# vs the TMA pipeline) and of the in-backward placement, with real compute.
set -x
mkdir -p gpurun_out
for v in 0 5; do
  AMSP_TAIL_VARIANT=$v timeout 900 python bench.py --compute gemm --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/r02_tail_v$v.json 2> gpurun_out/r02_tail_v$v.err
  echo "tail v$v rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/r02_tail_v$v.json').read().splitlines()[-1]); o=d['overlap']; print({k: o[k] for k in ('step_ms','compute_only_ms','compute_plus_optimizer_ms','exposed_frac')})"
done
timeout 900 python bench.py --compute gemm --no-e2e --no-cpu-baseline --steps 10 --optimizer-overlap 1 > gpurun_out/r02_tail_o1.json 2> gpurun_out/r02_tail_o1.err
python -c "import json; d=json.loads(open('gpurun_out/r02_tail_o1.json').read().splitlines()[-1]); o=d['overlap']; print({k: o[k] for k in ('step_ms','compute_only_ms','compute_plus_optimizer_ms','exposed_frac')})"
