mkdir -p gpurun_out
for w in weak1536_odf4 weak1536_odf8 weak1536_odf16 weak1536_odf32; do
python scripts/sweep.py "--workload $w --variant direct" "--workload $w --variant unfused" "--workload $w --variant C" 2>&1
done | tee gpurun_out/exp18.txt
python scripts/sweep.py '--launch per_block --variant unfused' '--launch per_block --variant B' '--launch per_block --variant direct' '--launch per_block --variant direct --graph 1' '--launch per_block --variant unfused --graph 1' -- --workload weak1536_odf8 2>&1 | tee -a gpurun_out/exp18.txt
