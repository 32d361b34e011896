mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --warmup 5 --steps 60 --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'], d['gpu_launches'])" 2>&1)"; }
run --grid 3072,1536,1536
J3D_PEERX_DIRECT=1 run --grid 3072,1536,1536
run --grid 3072,1536,1536 --launch persistent
run
run --launch persistent
run --workload fine384_odf64
run --workload fine384_odf64 --launch persistent
