# tile-configuration sweep: full parity once, parity subset + short bench per kind, then ncu captures
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/parity_full.log 2>&1
echo "full parity rc=$? $(tail -1 gpurun_out/parity_full.log)"
for k in ${KINDS:-0 1 2 3 4 5 6 7 8 9 10}; do
  J3D_TILE=$k timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear" > gpurun_out/sweep_parity_$k.log 2>&1
  echo "kind $k parity rc=$? $(tail -1 gpurun_out/sweep_parity_$k.log)"
  J3D_TILE=$k timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/sweep_bench_$k.log 2>&1
  echo "kind $k bench rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/sweep_bench_$k.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])" 2>&1)"
done
for k in ${NCU_KINDS:-}; do
  J3D_TILE=$k timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_plain_$k.log 2>&1 && \
  J3D_TILE=$k timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 3 -c 1 -o gpurun_out/prof_k$k python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_$k.log 2>&1
  echo "ncu kind $k rc=$?"
done
