# end-of-round check of the final commit state on one GPU (short: little budget left)
mkdir -p gpurun_out
timeout 120 python __graft_entry__.py smoke > gpurun_out/close_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/close_smoke.log
timeout 150 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/close_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/close_pytest.log
