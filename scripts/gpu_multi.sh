mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
J3D_MP_CASES=${CASES:-quick} timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/multi_$N.log 2>&1; echo "multi $N rc=$? $(tail -1 gpurun_out/multi_$N.log)"
for x in ${XCHG:-p2p nccl}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps ${STEPS:-30} --warmup 5 --exchange $x --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench_multi_${N}_$x.log 2>&1; echo "bench $N $x rc=$?"; tail -1 gpurun_out/bench_multi_${N}_$x.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('halo'), d['roofline']['frac'], d['clocks'], d['e2e']['value'] if d.get('e2e') else None)"
done
