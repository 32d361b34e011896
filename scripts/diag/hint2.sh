# TMA loads with an L2 evict_last policy (J3D_TMA_HINT=2) vs plain, per workload, alternating
S() { python scripts/sweep.py "$@"; }
for wl in "--workload fine384_odf64 --steps 100" "--workload fine768_odf64 --steps 100" "--workload small192_odf1 --steps 200" "--workload weak1536_odf8 --steps 30" "--workload weak1536_odf8 --variant C --steps 30" "--workload weak1536_odf8 --variant unfused --steps 30" "--workload weak1536_odf32 --steps 30" "--workload fine384_odf64 --launch batched --steps 100" "--steps 100"; do
  S "$wl" "J3D_TMA_HINT=2 $wl"
done
