timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tests/mp_worker.py persistent 2>&1 | grep -E "MP OK|FAIL|rror" | head -5
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k persistent 2>&1 | tail -1
