mkdir -p gpurun_out
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so" "J3D_TILE=14" "J3D_TILE=16" "J3D_TILE=12" "J3D_TILE=18" "J3D_TILE=15" "J3D_TILE=13" "J3D_TILE=4" "J3D_TILE=16 J3D_ZCHUNK=48" "J3D_TILE=12 J3D_ZCHUNK=48" "J3D_TILE=14 J3D_ZCHUNK=24" -- --workload fine384_odf64 --steps 200 --warmup 20
