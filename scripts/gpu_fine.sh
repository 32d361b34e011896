mkdir -p gpurun_out
A="--workload fine384_odf64 --steps 200 --warmup 20 --no-cpu --no-e2e"
python scripts/sweep.py \
 '--launch per_block --variant unfused' '--launch per_block --variant unfused --graph 1' \
 '--launch per_block --variant A' '--launch per_block --variant A --graph 1' \
 '--launch per_block --variant B' '--launch per_block --variant B --graph 1' \
 '--launch per_block --variant C' '--launch per_block --variant C --graph 1' \
 '--launch per_block --variant direct' '--launch per_block --variant direct --graph 1' \
 '--launch batched --variant unfused' '--launch batched --variant unfused --graph 1' \
 '--launch batched --variant C' '--launch batched --variant C --graph 1' \
 '--launch batched --variant direct' '--launch batched --variant direct --graph 1' \
 'J3D_TILE=11 --launch batched --variant direct' 'J3D_TILE=4 --launch batched --variant direct' 'J3D_TILE=7 --launch batched --variant direct' 'J3D_TILE=2 --launch batched --variant direct' \
 -- $A 2>&1 | tee gpurun_out/fine.txt
python scripts/sweep.py '--variant direct' '--variant unfused' '--variant C' -- --workload weak1536_odf8 --steps 30 --warmup 5 --no-cpu --no-e2e 2>&1 | tee gpurun_out/odf8.txt
python scripts/sweep.py '--variant direct' -- --workload small192_odf1 --steps 500 --warmup 20 --no-cpu --no-e2e 2>&1 | tee gpurun_out/small192.txt
