mkdir -p gpurun_out
nvidia-smi topo -m | head -5
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/multi.log 2>&1; echo "multi rc=$? $(tail -1 gpurun_out/multi.log)"
N=$(nvidia-smi -L | wc -l)
for x in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 30 --warmup 5 --exchange $x --no-cpu > gpurun_out/bench_multi_$x.log 2>&1; echo "bench $N $x rc=$?"; tail -1 gpurun_out/bench_multi_$x.log | cut -c1-1500
done
