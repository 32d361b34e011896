mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/parity_full.log 2>&1
echo "full parity rc=$? $(tail -1 gpurun_out/parity_full.log)"
for k in 1 4 9; do
  J3D_TILE=$k timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "shapes or config1 or linear or subnormal" > gpurun_out/sweep_parity_$k.log 2>&1
  echo "kind $k parity rc=$? $(tail -1 gpurun_out/sweep_parity_$k.log)"
done
python scripts/sweep.py \
  'J3D_TILE=11' 'J3D_TILE=11 J3D_ZCHUNK=96' 'J3D_TILE=4 J3D_ZCHUNK=96' 'J3D_TILE=10 J3D_ZCHUNK=96' 'J3D_TILE=12 J3D_ZCHUNK=96' \
  'J3D_TILE=9 J3D_ZCHUNK=96' 'J3D_TILE=1 J3D_ZCHUNK=64' 'J3D_TILE=2 J3D_ZCHUNK=64' 'J3D_TILE=7 J3D_ZCHUNK=64' 2>&1 | tee gpurun_out/exp3.txt
