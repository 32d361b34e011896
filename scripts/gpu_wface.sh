timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persistent.py -q -x 2>&1 | tail -1
for i in 1 2; do
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so" "J3D_X=0" "J3D_LIB=libjacobi3d_old.so --launch persistent" "--launch persistent" -- --workload fine384_odf64 --steps 200 --warmup 20
done
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so" "J3D_X=0" -- --workload weak1536_odf8 --steps 30 --warmup 5
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so --launch persistent" "--launch persistent" -- --workload fine768_odf64 --steps 200 --warmup 20
