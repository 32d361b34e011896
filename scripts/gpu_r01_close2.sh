# end-of-round: full GPU suite and the default N=1 bench line on the final commit state
mkdir -p gpurun_out
timeout 160 python -m pytest tests -m gpu -q > gpurun_out/close2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/close2_pytest.log
timeout 150 python bench.py > gpurun_out/close2_bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/close2_bench_n1.log
