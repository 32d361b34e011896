python scripts/sweep.py "J3D_TILE=4 J3D_ZCHUNK=8" "J3D_TILE=4 J3D_ZCHUNK=12" "J3D_TILE=4 J3D_ZCHUNK=16" "J3D_TILE=14 J3D_ZCHUNK=8" "J3D_TILE=14 J3D_ZCHUNK=12" "J3D_TILE=14 J3D_ZCHUNK=16" -- --workload small192_odf1 --steps 500 --warmup 20 --launch persistent
python scripts/sweep.py "J3D_TILE=4 J3D_ZCHUNK=12" "J3D_TILE=4 J3D_ZCHUNK=16" "J3D_TILE=4" -- --workload small192_odf1 --steps 500 --warmup 20
python scripts/sweep.py "J3D_ZCHUNK=12" "J3D_ZCHUNK=16" "J3D_X=0" -- --workload fine384_odf64 --steps 200 --warmup 20 --launch persistent
python scripts/sweep.py "J3D_ZCHUNK=32" "J3D_ZCHUNK=48" "J3D_X=0" -- --workload fine768_odf64 --steps 200 --warmup 20 --launch persistent
python scripts/sweep.py "J3D_ZCHUNK=48" "J3D_X=0" -- --workload weak1536_odf1 --steps 30 --warmup 5 --launch persistent
