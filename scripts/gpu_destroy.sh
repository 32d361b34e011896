N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tests/mp_worker.py persistent 2>&1 | grep -E "MP OK|FAIL|rror" | head -10
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k parity 2>&1 | tail -1
