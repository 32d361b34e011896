mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k every_tile_kind 2>&1 | tail -1
python scripts/sweep.py "J3D_TILE=12" "J3D_TILE=19" "J3D_TILE=12 --launch persistent" "J3D_TILE=19 --launch persistent" -- --workload fine384_odf64 --steps 200 --warmup 20
python scripts/sweep.py "J3D_X=0" "--launch persistent" -- --workload fine768_odf64 --steps 200 --warmup 20
