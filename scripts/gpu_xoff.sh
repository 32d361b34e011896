mkdir -p gpurun_out
J3D_LIB=libjacobi3d_x2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
bash scripts/ncu_sweep.sh "--workload fine384_odf64" "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_x2.so"
bash scripts/ncu_sweep.sh "--workload weak1536_odf1" "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_x2.so"
bash scripts/ncu_sweep.sh "--workload weak1536_odf8" "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_x2.so"
python scripts/sweep.py "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_x2.so" -- --workload fine384_odf64 --steps 200 --warmup 20
python scripts/sweep.py "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_x2.so" -- --workload weak1536_odf1 --steps 30 --warmup 5
python scripts/sweep.py "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_x2.so" -- --workload weak1536_odf8 --steps 30 --warmup 5
