python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.log 2>&1; echo bench rc=$?
python bench.py --gpus 1 --steps 100 --warmup 10 > gpurun_out/r02_bench_n1_100.log 2>&1; echo bench100 rc=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.log 2>&1; echo ref rc=$?
python bench.py --workload fine384_odf64 --steps 100 --warmup 10 --no-cpu --no-e2e > gpurun_out/r02_bench_fine384.log 2>&1; echo fine rc=$?
python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_launches.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:stencil -s 3 -c 1 -o /tmp/r02_stencil_default python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_default.log 2>&1; echo ncu1 rc=$?
python bench.py --workload fine384_odf64 --steps 100 --warmup 10 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stencil -s 1 -c 1 -o /tmp/r02_stencil_fine384 python bench.py --workload fine384_odf64 --steps 100 --warmup 10 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_fine.log 2>&1; echo ncu2 rc=$?
python bench.py --workload fine384_odf64 --launch batched --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stencil -s 3 -c 1 -o /tmp/r02_stencil_fine384_batched python bench.py --workload fine384_odf64 --launch batched --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_fine_b.log 2>&1; echo ncu3 rc=$?
for r in default fine384 fine384_batched; do
  ncu -i /tmp/r02_stencil_$r.ncu-rep --page raw --csv > gpurun_out/r02_stencil_$r.raw.csv 2>/dev/null
  ncu -i /tmp/r02_stencil_$r.ncu-rep --page details --csv > gpurun_out/r02_stencil_$r.details.csv 2>/dev/null
  ncu -i /tmp/r02_stencil_$r.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_stencil_$r.sass.csv 2>/dev/null
  gzip -9 gpurun_out/r02_stencil_$r.sass.csv
done
cp /tmp/r02_stencil_default.ncu-rep gpurun_out/
du -sh gpurun_out; ls -la gpurun_out
