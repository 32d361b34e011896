"""Write the committed ncu evidence for a round into profiles/.

    python scripts/write_profile.py --round r01 --workload weak1536_odf1 \
        --rep gpurun_out/prof_default.ncu-rep --launches gpurun_out/launches.csv --bench gpurun_out/bench_default.log

profiles/ncu_stencil_<round>.json : per-launch DRAM traffic of the stencil (bench.py reads `traffic`)
profiles/<round>_ncu_summary.md   : the metrics, the launch list shares and the bench line
"""
import argparse
import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in rows[1:]:
        out.append((r[ik], float(r[iv])))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--bench")
    ap.add_argument("--note", default="")
    ap.add_argument("--launch", required=True, help="launch mode of the captured run (bench.py --launch)")
    ap.add_argument("--variant", default="direct")
    ap.add_argument("--tile-kind", type=int, required=True, help="stats()['tile_kind'] of the captured run")
    ap.add_argument("--iters-per-launch", type=int, default=1)
    ap.add_argument("--alg-bytes", type=float, required=True, help="algorithmic bytes per captured launch")
    ap.add_argument("--name", default=None, help="file suffix (default: the round)")
    a = ap.parse_args()
    s = summary(a.rep)[0]
    rd = to_bytes(*s["dram__bytes_read.sum"])
    wr = to_bytes(*s["dram__bytes_write.sum"])
    dv, du = s["gpu__time_duration.sum"]
    dur_ms = float(dv) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}.get(du, 1.0)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    sys.path.insert(0, ROOT)
    import bench

    sha = bench.build_sha256()  # the sources the capture was taken with (bench.py checks it)
    js = {"round": a.round, "workload": a.workload, "launch": a.launch, "variant": a.variant,
          "tile_kind": a.tile_kind, "iters_per_launch": a.iters_per_launch, "build_sha256": sha,
          "kernel": s.get("kernel"), "traffic_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
          "dram_write_bytes": wr, "alg_bytes_per_launch": a.alg_bytes, "traffic_over_alg": (rd + wr) / a.alg_bytes,
          "ncu_duration_ms": dur_ms, "source": os.path.basename(a.rep),
          "metrics": {k: v for k, v in s.items() if k != "kernel"}}
    name = a.name or a.round
    with open(os.path.join(ROOT, "profiles", f"ncu_stencil_{name}.json"), "w") as f:
        json.dump(js, f, indent=1)
    md = [f"# {a.round}: ncu evidence for the stencil ({a.workload})", "", a.note, "",
          "## `ncu --set full --clock-control none` of one stencil launch", "", "| metric | value | unit |",
          "|---|---|---|"]
    for k, v in s.items():
        if k != "kernel":
            md.append(f"| {k} | {v[0]} | {v[1]} |")
    md += ["", f"kernel: `{s.get('kernel')}`", "",
           f"DRAM traffic per launch: read {rd/1e9:.3f} GB + write {wr/1e9:.3f} GB = {(rd+wr)/1e9:.3f} GB "
           f"(algorithmic {a.alg_bytes/1e9:.3f} GB: {(rd+wr)/a.alg_bytes:.4f}x)", ""]
    if a.launches:
        L = launches(a.launches)
        tot = sum(v for _, v in L)
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
               "| # | kernel | ms | share |", "|---|---|---|---|"]
        for i, (k, v) in enumerate(L):
            md.append(f"| {i} | `{k[:90]}` | {v/1e6:.3f} | {v/tot:.4f} |")
        st = sum(v for k, v in L if "stencil" in k)
        md += ["", f"stencil share of all launches: {st/tot:.4f} (includes setup launches of the run)", ""]
    if a.bench and os.path.exists(a.bench):
        line = [l for l in open(a.bench) if l.startswith("{")]
        if line:
            md += ["## bench.py line of the same build", "", "```", line[-1].strip(), "```", ""]
    with open(os.path.join(ROOT, "profiles", f"{name}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md))
    print("wrote profiles for", a.round)


if __name__ == "__main__":
    main()
