mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool ${TOOL:-memcheck} --target-processes all python __graft_entry__.py smoke > gpurun_out/sanitizer_${TOOL:-memcheck}.log 2>&1; echo "sanitizer ${TOOL:-memcheck} rc=$?"; tail -5 gpurun_out/sanitizer_${TOOL:-memcheck}.log
