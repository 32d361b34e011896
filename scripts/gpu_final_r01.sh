mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
run() { N=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'], (d.get('e2e') or {}).get('value'))" 2>&1)"; }
run 1
run 2
run 4
for N in 1 2 4; do
  run $N --workload small192_odf1 --steps 500 --warmup 20 --no-cpu --no-e2e
  run $N --workload small192_odf1 --steps 500 --warmup 20 --no-cpu --no-e2e --launch persistent
  run $N --workload fine384_odf64 --steps 200 --warmup 20 --no-cpu --no-e2e
  run $N --workload fine384_odf64 --steps 200 --warmup 20 --no-cpu --no-e2e --launch persistent
  run $N --workload fine768_odf64 --steps 200 --warmup 20 --no-cpu --no-e2e --launch persistent
done
