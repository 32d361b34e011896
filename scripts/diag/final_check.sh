python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke_final.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02_smoke_final.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_n1_final.log 2>&1; echo bench rc=$?; python3 -c "
import json; l=[x for x in open('gpurun_out/r02_bench_n1_final.log') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
print(d['value'], r['frac'], r['traffic'], r['traffic_source'], d['gpu_launches'], d['clocks'])"
for wl in "weak1536_odf8 --variant unfused" "weak1536_odf8"; do
  tag=$(echo $wl | tr ' ' '_' | tr -d '-')
  python bench.py --workload $wl --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_plain_$tag.log 2>&1 && ncu --set full --clock-control none -k regex:"stencil|copy_faces" -s 8 -c 4 -o /tmp/r02_$tag python bench.py --workload $wl --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_$tag.log 2>&1; echo ncu $tag rc=$?
  ncu -i /tmp/r02_$tag.ncu-rep --page raw --csv > gpurun_out/r02_odf8_$tag.raw.csv 2>/dev/null
done
du -sh gpurun_out
