mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
J3D_MP_CASES=quick timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "not fullsize" > gpurun_out/multi_$N.log 2>&1; echo "multi $N rc=$? $(tail -1 gpurun_out/multi_$N.log)"
grep -E "FAIL" gpurun_out/multi_$N.log | head -5 | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n$N.log | cut -c1-2500
