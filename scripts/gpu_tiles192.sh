mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k every_tile_kind 2>&1 | tail -2
run() { N=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'])" 2>&1)"; }
for T in 0 19 20 21; do
  J3D_TILE=$T run 4 --workload fine768_odf64 --steps 200 --warmup 20 --launch persistent
  J3D_TILE=$T run 2 --workload fine768_odf64 --steps 200 --warmup 20 --launch persistent
done
for T in 0 19 20 21; do
  J3D_TILE=$T run 1 --workload weak1536_odf1 --steps 30 --warmup 5
  J3D_TILE=$T run 1 --workload weak1536_odf8 --steps 30 --warmup 5
done
