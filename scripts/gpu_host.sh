mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tests/mp_worker.py debug > gpurun_out/mp_debug.log 2>&1; echo "debug rc=$?"
grep -E "FAIL|MP OK|Error" gpurun_out/mp_debug.log | head -10 | cut -c1-300
J3D_MP_CASES=quick timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/multi_$N.log 2>&1; echo "multi $N rc=$? $(tail -1 gpurun_out/multi_$N.log)"
grep -E "FAIL" gpurun_out/multi_$N.log | head -5 | cut -c1-400
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/b.log 2>&1; echo "bench $N $* rc=$? $(tail -1 gpurun_out/b.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], round(d['value']/d['n_gpus'],1), d['ms_per_step'], d.get('halo'), d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1)"; }
run --exchange host
run --exchange host --variant unfused
run --exchange host --overlap 1
run --exchange host --workload weak1536_odf8 --variant unfused --overlap 1
run --exchange p2p --workload small192_odf1 --steps 500
run --exchange host --workload small192_odf1 --steps 500
run --exchange nccl --workload small192_odf1 --steps 500
