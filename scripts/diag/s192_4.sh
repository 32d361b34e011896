# small192_odf1 (one 192^3 block per GPU, persistent): where do the 4-GPU microseconds go?
run() { n=$1; tag=$2; shift 2; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu --steps 400 --warmup 20 $ARGS > gpurun_out/r02_s192_${tag}.log 2>&1; python3 -c "
import json
l=[x for x in open('gpurun_out/r02_s192_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', d['ms_per_step'] if d else '', (d.get('halo') or {}) if d else '', d['roofline']['tile_kind'] if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
ARGS="--workload small192_odf1"
run 1 n1
run 1 n1_z12 J3D_ZCHUNK=12
run 4 n4
run 4 n4_z16 J3D_ZCHUNK=16
run 4 n4_z8 J3D_ZCHUNK=8
run 4 n4_k23 J3D_TILE=23
run 4 n4_k12 J3D_TILE=12
run 4 n4_k11 J3D_TILE=11
run 2 n2
ARGS="--workload small192_odf1 --launch batched"
run 4 n4_batched
ARGS="--workload small192_odf1 --launch batched --graph 1"
run 4 n4_batched_graph
ARGS="--workload small192_odf1 --grid 192,384,384 --odf 4"
run 1 n1_4blocks
