mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/parity_full.log 2>&1
echo "full parity rc=$? $(tail -1 gpurun_out/parity_full.log)"
for k in 1 2 3 5; do
J3D_TILE=$k timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear or subnormal" > gpurun_out/p_$k.log 2>&1; echo "kind $k parity rc=$? $(tail -1 gpurun_out/p_$k.log)"
done
python scripts/sweep.py 'J3D_TILE=0' 'J3D_TILE=1' 'J3D_TILE=6' 'J3D_TILE=8' 'J3D_TILE=3' 2>&1 | tee gpurun_out/exp11.txt
python scripts/sweep.py '--variant direct' '--variant unfused' -- --workload weak1536_odf8 2>&1 | tee -a gpurun_out/exp11.txt
python scripts/sweep.py 'J3D_TILE=2 --variant direct' 'J3D_TILE=4 --variant direct' 'J3D_TILE=2 --variant unfused' -- --workload fine384_odf64 --steps 200 --warmup 20 2>&1 | tee -a gpurun_out/exp11.txt
J3D_TILE=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_plain.log 2>&1 && \
J3D_TILE=0 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:stencil_tma -s 3 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__bytes|duration|inst_exec" | tr -s ' '
