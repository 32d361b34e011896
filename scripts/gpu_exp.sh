mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/parity_full.log 2>&1
echo "full parity rc=$? $(tail -1 gpurun_out/parity_full.log)"
for m in 1 3; do
J3D_TMA_HINT=$m timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear or subnormal" > gpurun_out/p_$m.log 2>&1; echo "tma $m parity rc=$? $(tail -1 gpurun_out/p_$m.log)"
done
python scripts/sweep.py '' 'J3D_TMA_HINT=1' 'J3D_TMA_HINT=2' 'J3D_TMA_HINT=3' 'J3D_TMA_HINT=3 J3D_STORE_HINT=1' 'J3D_TMA_HINT=1 J3D_STORE_HINT=1' '' 2>&1 | tee gpurun_out/exp10.txt
for m in 0 3; do
  J3D_TMA_HINT=$m timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_plain.log 2>&1 && \
  J3D_TMA_HINT=$m timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:stencil_tma -s 3 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__bytes|duration|hit_rate" | tr -s ' ' | sed "s/^/tma=$m /"
done
