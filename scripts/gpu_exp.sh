mkdir -p gpurun_out
for k in 15 16 17 18; do
J3D_TILE=$k timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear or subnormal or seeds" > gpurun_out/p_$k.log 2>&1; echo "kind $k parity rc=$? $(tail -1 gpurun_out/p_$k.log)"
done
python scripts/sweep.py 'J3D_TILE=14' 'J3D_TILE=15' 'J3D_TILE=16' 'J3D_TILE=18' 'J3D_TILE=14 --graph 1' -- --workload fine384_odf64 --steps 200 --warmup 20 2>&1 | tee gpurun_out/exp20.txt
python scripts/sweep.py 'J3D_TILE=0' 'J3D_TILE=17' -- --steps 20 2>&1 | tee -a gpurun_out/exp20.txt
python scripts/sweep.py 'J3D_TILE=4' 'J3D_TILE=17' 'J3D_TILE=0' -- --workload small192_odf1 --steps 500 --warmup 20 2>&1 | tee -a gpurun_out/exp20.txt
