mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/parity_full.log 2>&1
echo "full parity rc=$? $(tail -1 gpurun_out/parity_full.log)"
python scripts/sweep.py '' 'J3D_XSECTOR=0' '--graph 1' '--variant unfused' -- --workload fine384_odf64 --steps 200 --warmup 20 2>&1 | tee gpurun_out/exp17.txt
python scripts/sweep.py '--variant direct' 'J3D_XSECTOR=0 --variant direct' '--variant unfused' -- --workload weak1536_odf8 2>&1 | tee -a gpurun_out/exp17.txt
python scripts/sweep.py '' -- --workload small192_odf1 --steps 500 --warmup 20 2>&1 | tee -a gpurun_out/exp17.txt
