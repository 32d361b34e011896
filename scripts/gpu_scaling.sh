mkdir -p gpurun_out
run() { N=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'], d['gpu_launches'])" 2>&1)"; }
for N in 1 2 4; do
  run $N --workload strong1536_odf8 --steps 50 --warmup 5
  run $N --workload strong1536_odf8 --steps 50 --warmup 5 --launch persistent
done
for N in 1 2 4; do
  run $N --workload fine768_odf64 --steps 200 --warmup 20
  run $N --workload fine768_odf64 --steps 200 --warmup 20 --graph 1
  run $N --workload fine768_odf64 --steps 200 --warmup 20 --launch persistent
  run $N --workload fine768_odf64 --steps 200 --warmup 20 --launch per_block --variant unfused
  run $N --workload fine768_odf64 --steps 200 --warmup 20 --launch per_block --variant unfused --graph 1
done
for N in 1 2 4; do
  run $N --workload weak1536_odf8 --steps 30 --warmup 5
  run $N --workload weak1536_odf8 --steps 30 --warmup 5 --variant unfused
done
