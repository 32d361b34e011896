mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tests/mp_worker.py debug > gpurun_out/mp_debug.log 2>&1; echo "debug rc=$?"
grep -E "FAIL|MP OK|Error" gpurun_out/mp_debug.log | head -20
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 tests/mp_worker.py quick > gpurun_out/mp_quick.log 2>&1; echo "quick rc=$?"
grep -E "FAIL|MP OK" gpurun_out/mp_quick.log | cut -c1-300 | head -40
