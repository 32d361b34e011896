mkdir -p gpurun_out
J3D_TILE=21 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear or subnormal" > gpurun_out/sweep_parity_21.log 2>&1; echo "kind 21 parity rc=$? $(tail -1 gpurun_out/sweep_parity_21.log)"
python scripts/sweep.py '--variant direct' '--variant unfused' '--variant direct --graph 1' 'J3D_TILE=17 --variant direct' -- --workload fine384_odf64 --steps 200 --warmup 20 2>&1 | tee gpurun_out/exp9.txt
