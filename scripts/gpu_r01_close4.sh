# end-of-round, 2 GPUs: persistent cross-GPU launch, destroy race and thin-slab stress on the final state
mkdir -p gpurun_out
timeout 85 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tests/mp_worker.py persistent > gpurun_out/close4_mp2.log 2>&1; echo "mp rc=$?"; grep -E "MP OK|FAIL|rror" gpurun_out/close4_mp2.log | head -5
