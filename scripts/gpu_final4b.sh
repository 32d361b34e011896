mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --no-cpu > gpurun_out/bench_final_n4.log 2>&1; echo "bench4 rc=$?"; tail -1 gpurun_out/bench_final_n4.log | cut -c1-300
