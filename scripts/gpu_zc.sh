timeout 600 python -m pytest tests/test_gpu_persistent.py -q 2>&1 | tail -1
run() { N=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'])" 2>&1)"; }
mkdir -p gpurun_out
run 1 --workload fine384_odf64 --steps 200 --warmup 20
run 1 --workload small192_odf1 --steps 500 --warmup 20
run 1 --workload fine768_odf64 --steps 200 --warmup 20
run 4 --workload fine768_odf64 --steps 200 --warmup 20
run 4 --workload fine384_odf64 --steps 200 --warmup 20
