mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_2.log 2>&1; echo "pytest gpu rc=$? $(tail -1 gpurun_out/pytest_gpu_2.log)"
bash scripts/gpu_multi.sh 2>&1 | grep bench -A1
