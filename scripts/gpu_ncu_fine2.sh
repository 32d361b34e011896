mkdir -p gpurun_out
A="--workload fine384_odf64 --steps 20 --warmup 5 --no-cpu --no-e2e"
python bench.py $A > gpurun_out/fine_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 10 -c 1 -o gpurun_out/fine_direct_xg -f python bench.py $A > gpurun_out/ncu_fine.log 2>&1; echo "ncu rc=$?"
