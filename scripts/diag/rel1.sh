# persistent release: lane-0 acq_rel fence after the warp barrier (libjacobi3d_rel1.so, -DJ3D_REL1) vs all-lane SC fence
J3D_LIB=libjacobi3d_rel1.so timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -k "not fullsize" > gpurun_out/r02_rel1_multi.log 2>&1; echo multi rc=$?; tail -1 gpurun_out/r02_rel1_multi.log
run() { n=$1; tag=$2; lib=$3; shift 3; J3D_LIB=$lib python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu "$@" > gpurun_out/r02_rel_${tag}.log 2>&1; python3 -c "
import json
l=[x for x in open('gpurun_out/r02_rel_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', d['ms_per_step'] if d else '', round(d['value']/d['n_gpus']*16/6532.9,4) if d else '', (d.get('halo') or {}) if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
for rep in 1 2; do
for lib in libjacobi3d_rel1.so libjacobi3d.so; do
t=${lib%.so}; t=${t#libjacobi3d}; t=x${t}
run 4 s192_${t}_$rep $lib --workload small192_odf1 --steps 400 --warmup 20
run 2 s192n2_${t}_$rep $lib --workload small192_odf1 --steps 400 --warmup 20
run 4 f384_${t}_$rep $lib --workload fine384_odf64 --steps 100 --warmup 10
run 4 f768_${t}_$rep $lib --workload fine768_odf64 --steps 100 --warmup 10
done
done
