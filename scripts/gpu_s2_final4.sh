# 4-GPU box: the whole GPU suite at HEAD + smoke.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2700 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/fin_pytest4.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
