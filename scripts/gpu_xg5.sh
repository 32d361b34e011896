mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k every_tile_kind 2>&1 | tail -2
python scripts/sweep.py "J3D_TILE=12" "J3D_TILE=19" "J3D_TILE=20" "J3D_TILE=21" "J3D_TILE=22" "J3D_TILE=12 --launch persistent" "J3D_TILE=19 --launch persistent" "J3D_TILE=20 --launch persistent" "J3D_TILE=21 --launch persistent" "J3D_TILE=22 --launch persistent" -- --workload fine384_odf64 --steps 200 --warmup 20
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so" "J3D_X=1" "J3D_LIB=libjacobi3d_old.so" "J3D_X=1" -- --workload weak1536_odf1 --steps 100 --warmup 10
