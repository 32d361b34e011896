python scripts/sweep.py "J3D_X=0" "J3D_ZCHUNK=32" "J3D_ZCHUNK=48" -- --workload fine384_odf64 --steps 200 --warmup 20
python scripts/sweep.py "J3D_X=0" "J3D_ZCHUNK=32" "J3D_ZCHUNK=64" -- --workload fine768_odf64 --steps 200 --warmup 20
