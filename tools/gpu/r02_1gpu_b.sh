# 1 GPU: the gradient-ring / sync-emulation tests, the default bench line, its
# ncu launch list, and ncu --set full of every default kernel (summaries).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sync_emulation_gpu.py tests/test_engine_gpu.py -q -p no:cacheprovider -k "ring or synced or scheduler" > gpurun_out/r02_pytest_ring.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02_pytest_ring.log
timeout 900 python bench.py > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r02_bench_n1.json; tail -3 gpurun_out/r02_bench_n1.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_n1.csv python bench.py > gpurun_out/r02_ncu_launches_run.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py launches gpurun_out/r02_launches_n1.csv > gpurun_out/r02_launches_n1_summary.json 2>&1; head -40 gpurun_out/r02_launches_n1_summary.json
bash tools/gpu/ncu_heads.sh
for f in gpurun_out/ncu/*.json; do echo "== $f"; python -c "import json,sys; d=json.load(open('$f')); [print({k: x.get(k) for k in ('kernel','gpu__time_duration.sum','dram_traffic_bytes','traffic_over_algorithmic','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active')}) for x in d]" 2>&1 | head -5; done
du -sh gpurun_out
