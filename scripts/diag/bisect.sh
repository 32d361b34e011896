run() { dir=$1; tag=$2; shift 2; (cd $dir && python bench.py --no-e2e --no-cpu "$@" > /root/repo/gpurun_out/r02_bis_${tag}.log 2>&1); python3 -c "
import json
l=[x for x in open('/root/repo/gpurun_out/r02_bis_${tag}.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('${tag}', d['value'] if d else 'FAIL', d['clocks'].get('sm_mhz') if d else '')
"; }
for rep in 1 2; do
for b in _r01 _b_c81cf87 _b_bdca31d _b_34660d7 _b_5b417fd .; do
run /root/repo/$b fine768_${b}_$rep --workload fine768_odf64 --steps 100 --warmup 10
run /root/repo/$b small192_${b}_$rep --workload small192_odf1 --steps 200 --warmup 10
done
done
