mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k fullsize > gpurun_out/multi_full_$N.log 2>&1; echo "multi fullsize $N rc=$? $(tail -1 gpurun_out/multi_full_$N.log)"
grep -E "Error|assert" gpurun_out/multi_full_$N.log | head -5 | cut -c1-300
if [ "$N" = "4" ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --workload strong3072_odf2 > gpurun_out/b_strong.log 2>&1; echo "strong3072 rc=$?"; tail -1 gpurun_out/b_strong.log | cut -c1-400
fi
