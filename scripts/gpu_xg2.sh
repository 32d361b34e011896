mkdir -p gpurun_out
for i in 1 2; do
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so" "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_nf.so" -- --workload fine384_odf64 --steps 200 --warmup 20
done
python scripts/sweep.py "J3D_LIB=libjacobi3d_old.so" "J3D_LIB=libjacobi3d.so" "J3D_LIB=libjacobi3d_nf.so" -- --workload weak1536_odf8 --steps 30 --warmup 5
