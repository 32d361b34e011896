mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/parity_full.log 2>&1
echo "full parity rc=$? $(tail -1 gpurun_out/parity_full.log)"
for k in 16 17; do
J3D_TILE=$k timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear or subnormal" > gpurun_out/sweep_parity_$k.log 2>&1; echo "kind $k parity rc=$? $(tail -1 gpurun_out/sweep_parity_$k.log)"
done
python scripts/sweep.py '--variant direct' 2>&1 | tee gpurun_out/exp8.txt
python scripts/sweep.py '--variant direct' '--variant unfused' 'J3D_TILE=16 --variant direct' -- --workload weak1536_odf8 2>&1 | tee -a gpurun_out/exp8.txt
python scripts/sweep.py '--variant direct' '--variant unfused' '--variant direct --graph 1' -- --workload fine384_odf64 --steps 200 --warmup 20 2>&1 | tee -a gpurun_out/exp8.txt
