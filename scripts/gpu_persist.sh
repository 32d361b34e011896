mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -15
python scripts/sweep.py "--launch batched" "--launch persistent" -- --workload fine384_odf64 --steps 200 --warmup 20
python scripts/sweep.py "--launch batched" "--launch persistent" "--launch batched --graph 1" -- --workload small192_odf1 --steps 500 --warmup 20
python scripts/sweep.py "--launch batched" "--launch persistent" -- --workload weak1536_odf1 --steps 30 --warmup 5
python scripts/sweep.py "--launch batched" "--launch persistent" -- --workload weak1536_odf8 --steps 30 --warmup 5
