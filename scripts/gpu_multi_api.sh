mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
J3D_MP_CASES=quick timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "not fullsize" > gpurun_out/multi_$N.log 2>&1; echo "multi $N rc=$? $(tail -1 gpurun_out/multi_$N.log)"
grep -E "FAIL|Error" gpurun_out/multi_$N.log | head -5 | cut -c1-300
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --warmup 20 --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'])" 2>&1)"; }
run --steps 200 --workload fine384_odf64
run --steps 200 --workload fine384_odf64 --graph 1
