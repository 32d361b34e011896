# wavefront slab order: z-chunk length across GPUs (this build; J3D_ZCHUNK = planes per chunk)
run() { n=$1; tag=$2; shift 2; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu $ARGS > gpurun_out/r02_wf2_${tag}.log 2>&1; python3 -c "
import json
l=[x for x in open('gpurun_out/r02_wf2_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', d['ms_per_step'] if d else '', round(d['value']/d['n_gpus']*16/6532.9,4) if d else '', (d.get('halo') or {}) if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
ARGS="--workload small192_odf1 --steps 400 --warmup 20"
run 4 s192_def
run 4 s192_z8 J3D_ZCHUNK=8
run 4 s192_z16 J3D_ZCHUNK=16
run 4 s192_z24 J3D_ZCHUNK=24
run 4 s192_old J3D_LIB=libjacobi3d_old.so
run 2 s192n2_z16 J3D_ZCHUNK=16
run 2 s192n2_z24 J3D_ZCHUNK=24
ARGS="--workload fine384_odf64 --steps 100 --warmup 10"
run 4 f384_def
run 4 f384_z32 J3D_ZCHUNK=32
run 4 f384_z24 J3D_ZCHUNK=24
ARGS="--workload fine768_odf64 --steps 100 --warmup 10"
run 4 f768_def
run 4 f768_z32 J3D_ZCHUNK=32
run 4 f768_z48 J3D_ZCHUNK=48
ARGS="--workload small192_odf1 --steps 400 --warmup 20"
run 4 s192_def_b
