# end-of-round: fine-grained (persistent) bench line and the reference (CPU oracle) arm on the final state
mkdir -p gpurun_out
timeout 100 python bench.py --workload fine384_odf64 > gpurun_out/close3_fine.log 2>&1; echo "fine rc=$?"; tail -1 gpurun_out/close3_fine.log
timeout 80 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/close3_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/close3_ref.log
