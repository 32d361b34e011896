mkdir -p gpurun_out
for cfg in "J3D_TILE=0" "J3D_TILE=0 J3D_ZCHUNK=1536" "J3D_TILE=0 J3D_ZCHUNK=384" "J3D_TILE=0 J3D_TILE_ORDER=1" "J3D_TILE=6" "J3D_TILE=3" "J3D_TILE=1"; do
  env $cfg timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_plain.log 2>&1 && \
  env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:stencil_tma -s 3 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__bytes|duration" | tr -s ' ' | sed "s/^/$cfg /"
done
