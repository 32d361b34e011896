mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --warmup 5 --steps 60 --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'])" 2>&1)"; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tests/mp_worker.py full 2>&1 | grep -E "MP OK|FAIL|Error" | head
run --grid 3072,1536,1536
run --grid 3072,1536,1536 --exchange nccl
run --grid 3072,1536,1536 --exchange host --overlap 1
run --grid 3072,1536,1536 --overlap 1
