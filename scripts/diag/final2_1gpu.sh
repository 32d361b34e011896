python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu_full.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02_pytest_gpu_full.log
bash scripts/diag/final_ncu.sh
