timeout 900 python -m pytest tests/test_gpu_parity.py -q -k plan_bytes 2>&1 | tail -1
python scripts/sweep.py "J3D_X=0" "J3D_ZCHUNK=192" "J3D_ZCHUNK=384" "--launch persistent" "J3D_ZCHUNK=192 --launch persistent" "J3D_ZCHUNK=384 --launch persistent" "J3D_X=0" -- --workload weak1536_odf1 --steps 30 --warmup 5
