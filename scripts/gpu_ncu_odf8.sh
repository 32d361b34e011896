mkdir -p gpurun_out
A="--workload weak1536_odf8 --steps 3 --warmup 3 --no-cpu --no-e2e"
python bench.py $A > /dev/null 2>&1; echo "plain rc=$?"
python bench.py $A --variant unfused > /dev/null 2>&1; echo "plain2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 5 -c 1 -o gpurun_out/prof_odf8_direct -f python bench.py $A > gpurun_out/ncu_a.log 2>&1; echo "a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 5 -c 1 -o gpurun_out/prof_odf8_unfused -f python bench.py $A --variant unfused > gpurun_out/ncu_b.log 2>&1; echo "b rc=$?"
B="--workload fine384_odf64 --steps 20 --warmup 3 --no-cpu --no-e2e --launch persistent"
python bench.py $B > /dev/null 2>&1; echo "plain3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches_persistent.csv python bench.py $B > gpurun_out/ncu_c.log 2>&1; echo "c rc=$?"
