mkdir -p gpurun_out
run() { N=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'])" 2>&1)"; }
for O in 1 2 4 8 16; do
  run 4 --workload strong3072_odf2 --odf $O --steps 30 --warmup 5
  run 4 --workload strong3072_odf2 --odf $O --steps 30 --warmup 5 --launch persistent
done
