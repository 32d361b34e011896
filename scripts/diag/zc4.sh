run() { n=$1; tag=$2; wl=$3; shift 3; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu --workload $wl --steps 100 --warmup 10 > gpurun_out/r02_zc4_${tag}.log 2>&1; python3 -c "
import json
l=[x for x in open('gpurun_out/r02_zc4_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', round(d['value']/d['n_gpus']*16/6532.9,4) if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
run 4 f384_def fine384_odf64
run 4 f384_z32 fine384_odf64 J3D_ZCHUNK=32
run 4 f384_z24 fine384_odf64 J3D_ZCHUNK=24
run 4 f768_z24 fine768_odf64 J3D_ZCHUNK=24
run 4 f768_z32 fine768_odf64 J3D_ZCHUNK=32
run 4 s192_def small192_odf1
run 4 s192_z24 small192_odf1 J3D_ZCHUNK=24
run 4 s192_z12 small192_odf1 J3D_ZCHUNK=12
run 2 f384_def2 fine384_odf64
run 2 f384_z32_2 fine384_odf64 J3D_ZCHUNK=32
run 2 f768_def2 fine768_odf64
run 2 f768_z32_2 fine768_odf64 J3D_ZCHUNK=32
python scripts/sweep.py 'J3D_LIB=libjacobi3d.so --workload weak1536_odf8 --steps 50' 'J3D_LIB=libjacobi3d_m1w.so --workload weak1536_odf8 --steps 50' 'J3D_LIB=libjacobi3d.so --workload weak1536_odf32 --steps 50' 'J3D_LIB=libjacobi3d_m1w.so --workload weak1536_odf32 --steps 50' 'J3D_LIB=libjacobi3d.so --workload weak1536_odf32 --variant C --steps 50' 'J3D_LIB=libjacobi3d_m1w.so --workload weak1536_odf32 --variant C --steps 50' 'J3D_LIB=libjacobi3d.so --workload fine768_odf64 --steps 100' 'J3D_LIB=libjacobi3d_m1w.so --workload fine768_odf64 --steps 100'
