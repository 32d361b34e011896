# persistent z-chunk: one 96-plane chunk per 96^3 block vs the default rule (48)
mkdir -p gpurun_out
for zc in 0 96 64; do
  if [ $zc = 0 ]; then unset J3D_ZCHUNK; else export J3D_ZCHUNK=$zc; fi
  timeout 45 python bench.py --workload fine384_odf64 --no-cpu --no-e2e --steps 200 > gpurun_out/zc_$zc.log 2>&1
  echo "zc=$zc rc=$? $(tail -1 gpurun_out/zc_$zc.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])' 2>&1)"
done
