"""Run bench.py under several env/argument settings and print one summary line each.

    python scripts/sweep.py 'J3D_TILE=1' 'J3D_TILE=9 J3D_ZCHUNK=64' ... [-- extra bench args]
"""
import json
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    argv = sys.argv[1:]
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    base = ["--steps", "20", "--warmup", "5", "--no-cpu", "--no-e2e"] + extra
    for setting in argv:
        env = dict(os.environ)
        args = list(base)
        for tok in shlex.split(setting):
            if "=" in tok and not tok.startswith("--"):
                k, v = tok.split("=", 1)
                env[k] = v
            else:
                args.append(tok)
        try:
            p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env, capture_output=True,
                               text=True, timeout=600)
            line = [l for l in p.stdout.strip().splitlines() if l.startswith("{")]
            if p.returncode != 0 or not line:
                print(f"{setting:40s} FAILED rc={p.returncode} {p.stderr.strip()[-300:]}", flush=True)
                continue
            d = json.loads(line[-1])
            r = d.get("roofline") or {}
            print(f"{setting:40s} {d['value']:9.2f} GLUPS {d['ms_per_step']:8.3f} ms  frac={r.get('frac')}  "
                  f"clk={d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}", flush=True)
        except subprocess.TimeoutExpired:
            print(f"{setting:40s} TIMEOUT", flush=True)


if __name__ == "__main__":
    main()
