# usage: bash scripts/ncu_sweep.sh "<bench args>" "ENV=.. ENV2=.." ...   (one ncu metric pass per setting)
mkdir -p gpurun_out
ARGS="$1"; shift
for S in "$@"; do
  env $S timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,sm__cycles_active.avg --clock-control none -k regex:stencil_tma -s 2 -c 1 --csv python bench.py $ARGS --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_sweep.csv 2>/dev/null
  python - "$S" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/ncu_sweep.csv")) if len(r) > 10 and (r[0] == "ID" or r[0].isdigit())]
h = rows[0]; iN = h.index("Metric Name"); iV = h.index("Metric Value"); iU = h.index("Metric Unit")
m = {r[iN]: (r[iV], r[iU]) for r in rows[1:]}
def g(k): return m.get(k, ("?", ""))
print(f"{sys.argv[1]:40s} t={g('gpu__time_duration.sum')} rd={g('dram__bytes_read.sum')} wr={g('dram__bytes_write.sum')} texrd={g('lts__t_sectors_srcunit_tex_op_read.sum')[0]} hit={g('lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum')[0]} act={g('sm__cycles_active.avg')[0]}", flush=True)
PY
done
