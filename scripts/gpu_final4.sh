mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest gpu (4 GPUs visible) rc=$? $(tail -1 gpurun_out/pytest_gpu4.log)"
grep -E "FAIL|Error" gpurun_out/pytest_gpu4.log | head -5 | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/bench_n4.log 2>&1; echo "bench 4 rc=$?"; tail -1 gpurun_out/bench_n4.log | cut -c1-3000
