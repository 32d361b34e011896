# round 1 (git 7b0adda, built in _r01/) vs this build, same box, alternating
run() { dir=$1; n=$2; tag=$3; shift 3; (cd $dir && python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --no-e2e --no-cpu "$@" > /root/repo/gpurun_out/r02_ab_${tag}.log 2>&1); python3 -c "
import json,sys
l=[x for x in open('/root/repo/gpurun_out/r02_ab_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', d['ms_per_step'] if d else '', d['clocks'].get('sm_mhz') if d else '')
"; }
for rep in 1 2; do
run /root/repo 4 r02_fine768_$rep --workload fine768_odf64 --steps 100 --warmup 10
run /root/repo/_r01 4 r01_fine768_$rep --workload fine768_odf64 --steps 100 --warmup 10
done
run /root/repo 4 r02_fine384 --workload fine384_odf64 --steps 100 --warmup 10
run /root/repo/_r01 4 r01_fine384 --workload fine384_odf64 --steps 100 --warmup 10
run /root/repo 4 r02_small192 --workload small192_odf1 --steps 200 --warmup 10
run /root/repo/_r01 4 r01_small192 --workload small192_odf1 --steps 200 --warmup 10
run /root/repo 4 r02_weak1536 --steps 30 --warmup 5
run /root/repo/_r01 4 r01_weak1536 --steps 30 --warmup 5
run /root/repo 1 r02_fine768_1 --workload fine768_odf64 --steps 100 --warmup 10
run /root/repo/_r01 1 r01_fine768_1 --workload fine768_odf64 --steps 100 --warmup 10
