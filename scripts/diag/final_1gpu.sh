set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/r02_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu_full.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02_pytest_gpu_full.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/r02_bench_n1.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/r02_bench_ref.log
python bench.py --workload fine384_odf64 --steps 100 --warmup 10 --no-cpu --no-e2e > gpurun_out/r02_bench_fine384.log 2>&1; echo fine rc=$?; tail -1 gpurun_out/r02_bench_fine384.log
python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_launches.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:stencil -s 3 -c 1 -o gpurun_out/r02_stencil_default python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_default.log 2>&1; echo ncu1 rc=$?
python bench.py --workload fine384_odf64 --steps 10 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stencil -s 1 -c 1 -o gpurun_out/r02_stencil_fine384 python bench.py --workload fine384_odf64 --steps 10 --warmup 3 --repeats 1 --no-cpu --no-e2e > gpurun_out/r02_ncu_fine.log 2>&1; echo ncu2 rc=$?
