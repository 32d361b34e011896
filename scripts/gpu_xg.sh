mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
bash scripts/ncu_sweep.sh "--workload fine384_odf64" "J3D_X=0"
bash scripts/ncu_sweep.sh "--workload weak1536_odf1" "J3D_X=0"
python scripts/sweep.py "--launch batched" "--launch persistent" -- --workload fine384_odf64 --steps 200 --warmup 20
python scripts/sweep.py "--launch batched" -- --workload weak1536_odf1 --steps 30 --warmup 5
python scripts/sweep.py "--launch batched" -- --workload weak1536_odf8 --steps 30 --warmup 5
