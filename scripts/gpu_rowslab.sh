mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tests/mp_worker.py persistent 2>&1 | grep -E "MP OK|FAIL|Error|error" | head -20
run() { N=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'])" 2>&1)"; }
for N in 1 2 4; do
  run $N --steps 60 --warmup 5
  run $N --steps 60 --warmup 5 --launch persistent
done
run 4 --workload small192_odf1 --steps 500 --warmup 20 --launch persistent
run 4 --workload fine384_odf64 --steps 200 --warmup 20 --launch persistent
run 4 --workload fine768_odf64 --steps 200 --warmup 20 --launch persistent
run 1 --workload fine384_odf64 --steps 200 --warmup 20 --launch persistent
run 1 --workload small192_odf1 --steps 500 --warmup 20 --launch persistent
