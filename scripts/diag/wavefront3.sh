# persistent slab order across GPUs (J3D_WAVE): 0 exterior last only (round-2 order), 1 deepest first, 2 exterior first
run() { n=$1; tag=$2; shift 2; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu $ARGS > gpurun_out/r02_wf3_${tag}.log 2>&1; python3 -c "
import json
l=[x for x in open('gpurun_out/r02_wf3_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', d['ms_per_step'] if d else '', round(d['value']/d['n_gpus']*16/6532.9,4) if d else '', (d.get('halo') or {}) if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
for w in 0 1 2; do
ARGS="--workload small192_odf1 --steps 400 --warmup 20"
run 4 s192_w$w J3D_WAVE=$w
run 2 s192n2_w$w J3D_WAVE=$w
ARGS="--workload fine384_odf64 --steps 100 --warmup 10"
run 4 f384_w$w J3D_WAVE=$w
run 4 f384_z32_w$w J3D_WAVE=$w J3D_ZCHUNK=32
ARGS="--workload fine768_odf64 --steps 100 --warmup 10"
run 4 f768_w$w J3D_WAVE=$w
run 4 f768_z48_w$w J3D_WAVE=$w J3D_ZCHUNK=48
done
