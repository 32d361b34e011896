run() { n=$1; tag=$2; shift 2; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu --workload fine768_odf64 --steps 100 --warmup 10 > gpurun_out/r02_f768_${tag}.log 2>&1; python3 -c "
import json
l=[x for x in open('gpurun_out/r02_f768_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', round(d['value']/d['n_gpus']*16/6532.9,4) if d else '', d['roofline']['tile_kind'] if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
run 4 k21 J3D_TILE=21
run 4 k26 J3D_TILE=26
run 4 k0 J3D_TILE=0
run 4 k21_z48 J3D_TILE=21 J3D_ZCHUNK=48
run 4 k26_z48 J3D_TILE=26 J3D_ZCHUNK=48
run 4 k21_z32 J3D_TILE=21 J3D_ZCHUNK=32
run 4 k21b J3D_TILE=21
run 1 n1_k21 J3D_TILE=21
run 1 n1_k26 J3D_TILE=26
run 2 n2_k21 J3D_TILE=21
run 2 n2_k26 J3D_TILE=26
