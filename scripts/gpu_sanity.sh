timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py --workload fine384_odf64 --steps 100 --warmup 10 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['launch'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['gpu_launches'])"
python bench.py --workload small192_odf1 --steps 300 --warmup 10 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['launch'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['gpu_launches'])"
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['launch'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['gpu_launches'])"
