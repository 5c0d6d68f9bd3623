set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sync_emulation_gpu.py -q -p no:cacheprovider -k "zeropp or push" > gpurun_out/r02_pytest_push2.log 2>&1; echo "sync rc=$?"; tail -4 gpurun_out/r02_pytest_push2.log
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "push" > gpurun_out/r02_pytest_push2_mp.log 2>&1; echo "mp rc=$?"; tail -4 gpurun_out/r02_pytest_push2_mp.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29821 bench.py --gpus 4 --model llama-13b --plan p=4x1,g=4x1,os=4x1,p2=2x1 --no-overlap --no-e2e --no-cpu-baseline --no-grad-ring > gpurun_out/r02_zeropp_push_n4.json 2> gpurun_out/r02_zeropp_push_n4.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02_zeropp_push_n4.json').read().splitlines()[-1]); r=d['roofline']; print(d['ms_per_step'], r['step_breakdown_ms'], r.get('frac_of_phase_bound'))"
