#!/usr/bin/env python
"""Jacobi3D benchmark (BASELINE.json metric: GLUPS and ms/iter, HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one Jacobi iteration of the whole hot path over the job's grid:
the stencil update of every block plus the pack/exchange/unpack of every face
(fused into the update for the default "direct" variant), on synthetic
hash-random fp64 data (seed 20220223, Dirichlet boundary 1.0).

Default workload (BASELINE.json configs[1], the one the metric is quoted on):
weak scaling, 1536^3 cells per GPU, ODF=1, batched launch (one stencil launch
per iteration).  The small and fine-grained workloads default to the persistent
launch (one stencil launch per timed region, --launch overrides).  Rank 0
prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Jacobi3D GLUPS and ms/iter at 1/2/4/8 B200; achieved HBM GB/s vs peak"
SEED = 20220223
BYTES_PER_LUP = 16.0  # algorithmic HBM bytes per lattice-site update (read u^n + write u^{n+1}, fp64)

L2_BYTES = 126.5e6  # B200 L2 (both dies)

# name -> weak (per-GPU dims) or strong (global dims), odf
WORKLOADS = {
    # configs[1]: weak scaling, 1536^3 per GPU, ODF=1
    "weak1536_odf1": dict(kind="weak", per_gpu=(1536, 1536, 1536), odf=1),
    # configs[2]: weak scaling with overdecomposition
    "weak1536_odf4": dict(kind="weak", per_gpu=(1536, 1536, 1536), odf=4),
    "weak1536_odf8": dict(kind="weak", per_gpu=(1536, 1536, 1536), odf=8),
    "weak1536_odf16": dict(kind="weak", per_gpu=(1536, 1536, 1536), odf=16),
    "weak1536_odf32": dict(kind="weak", per_gpu=(1536, 1536, 1536), odf=32),
    # configs[3]: strong scaling 3072^3 (needs >= 4 GPUs: 464 GB double-buffered)
    "strong3072_odf2": dict(kind="strong", global_=(3072, 3072, 3072), odf=2),
    # SURVEY 8(d) config 4': strong scaling that reaches 1 GPU, 1536^3 global, ODF 8
    "strong1536_odf8": dict(kind="strong", global_=(1536, 1536, 1536), odf=8),
    # configs[4]: fine-grained, 768^3 global (8 GPUs x ODF 64 = 96^3 blocks)
    "fine768_odf64": dict(kind="strong", global_=(768, 768, 768), odf=64, launch="persistent"),
    # configs[4] per GPU: 384^3 per GPU with ODF 64 = the 96^3 blocks of 768^3 on 8 GPUs
    "fine384_odf64": dict(kind="weak", per_gpu=(384, 384, 384), odf=64, launch="persistent"),
    # the paper's small weak-scaling problem (192^3 per node)
    "small192_odf1": dict(kind="weak", per_gpu=(192, 192, 192), odf=1, launch="persistent"),
    # configs[0]: the small oracle-checkable case
    "small64_odf8": dict(kind="strong", global_=(64, 64, 64), odf=8),
}


def weak_global(per_gpu, n):
    """Global grid for weak scaling: the surface-minimising GPU grid over n
    (1,1,1)/(1,1,2)/(1,2,2)/(2,2,2) times the per-GPU block."""
    grids = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}
    if n not in grids:
        raise SystemExit(f"weak scaling supports 1/2/4/8 GPUs, got {n}")
    g = grids[n]
    return tuple(p * k for p, k in zip(per_gpu, g))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            t = [x.strip() for x in line.split(",")]
            if len(t) < 8:
                continue
            try:
                sm.append(float(t[1]))
                mx.append(float(t[2]))
            except ValueError:
                continue
            for nm, v in zip(names, t[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_sha256():
    """sha256 over the library's sources and build script (csrc/, include/, build.py):
    ties an ncu capture to the code it measured.  (Not the .so itself: nvcc output
    is not bit-reproducible, so every rebuild of the same sources hashes differently.)"""
    import glob
    import hashlib

    h = hashlib.sha256()
    pk = os.path.join(ROOT, "paper_2202_11819_b200")
    files = sorted(glob.glob(os.path.join(pk, "csrc", "*")) + glob.glob(os.path.join(ROOT, "include", "*.h")) +
                   [os.path.join(pk, "build.py")])
    for f in files:
        h.update(os.path.relpath(f, ROOT).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def traffic_from_profiles(workload, launch, variant, tile_kind, steps):
    """dram__bytes_read.sum + dram__bytes_write.sum per stencil launch from a
    committed ncu --set full summary (profiles/ncu_stencil_*.json) -- only one
    captured from THIS build (sha256 of the library's sources) with the same workload,
    launch mode, variant and tile kind (and, for the persistent launch, the
    same iterations per launch); otherwise None and the reason."""
    import glob

    sha = build_sha256()
    why = "no committed ncu capture for this workload"
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_stencil_*.json"))):
        try:
            with open(p) as f:
                d = json.load(f)
        except Exception:
            continue
        if d.get("workload") != workload or not d.get("traffic_bytes_per_launch"):
            continue
        want = {"build_sha256": sha, "launch": launch, "variant": variant, "tile_kind": tile_kind}
        if launch == "persistent":
            want["iters_per_launch"] = steps
        bad = [k for k, v in want.items() if d.get(k) != v]
        if bad:
            why = f"{os.path.basename(p)}: {', '.join(bad)} differ from this run"
            continue
        return d, os.path.basename(p)
    return None, why


def cpu_baseline(workload_grid, budget_s=12.0):
    """The oracle as it stands, on the host cores: a bounded sample of the same
    workload (an x-y-full slab of the global grid), timed over whole sweeps."""
    import numpy as np

    from oracle import core

    gx, gy, gz = workload_grid
    slab = max(4, min(gz, 64))
    U = core.init(gx, gy, slab, core.INIT_HASH, seed=SEED)
    V = U.copy()
    core.sweep_owned_timing(U, V)  # warm-up (page-in)
    n, t0 = 0, time.perf_counter()
    while True:
        core.sweep_owned_timing(U, V)
        U, V = V, U
        n += 1
        el = time.perf_counter() - t0
        if el > budget_s or n >= 1000:
            break
    lups = gx * gy * slab * n
    el_all = el
    # the same sweep on one core (the oracle at all cores and at 1 core)
    cores = core.threads()
    core.set_threads(1)
    n1, t1 = 0, time.perf_counter()
    try:
        while True:
            core.sweep_owned_timing(U, V)
            U, V = V, U
            n1 += 1
            el1 = time.perf_counter() - t1
            if el1 > budget_s / 4 or n1 >= 1000:
                break
    finally:
        core.set_threads(cores)
    del U, V
    return {"value": lups / el_all / 1e9, "unit": "GLUPS", "cores": cores, "kind": "oracle",
            "value_1core": gx * gy * slab * n1 / el1 / 1e9, **host_cpu(),
            "sample": f"{n} full sweeps of a {gx}x{gy}x{slab} slab of the workload (hash init, seed {SEED}), "
                      f"{el_all:.1f} s on {cores} threads; {n1} sweeps in {el1:.1f} s on 1 thread"}


def host_cpu():
    """The host the oracle ran on (nproc and the CPU model)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"cpu_model": model, "nproc": aff or os.cpu_count(), "cpu_count": os.cpu_count()}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="weak1536_odf1", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="direct")
    ap.add_argument("--launch", default=None,
                    help="per_block | batched | persistent (default: the workload's measured best; "
                         "batched for the 1536^3 configs, persistent for the small / fine-grained ones)")
    ap.add_argument("--graph", type=int, default=0)
    ap.add_argument("--exchange", default="auto")
    ap.add_argument("--overlap", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--grid", default=None, help="override global grid gx,gy,gz")
    ap.add_argument("--odf", type=int, default=None)
    ap.add_argument("--repeats", type=int, default=3,
                    help="timed regions of exactly K steps each; value = their mean (PAPER.md L583-584: "
                         "averages of 3 runs)")
    return ap.parse_args()


def main():
    a = parse()
    if a.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus:
        if world == 1 and a.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun --nproc-per-node N")
    n = a.gpus
    wl = dict(WORKLOADS[a.workload])
    grid = weak_global(wl["per_gpu"], n) if wl["kind"] == "weak" else wl["global_"]
    if a.grid:
        grid = tuple(int(x) for x in a.grid.split(","))
    odf = a.odf or wl["odf"]
    if a.launch is None:  # the persistent launch exists for the direct variant only
        a.launch = wl.get("launch", "batched") if a.variant == "direct" else "batched"
    cfg_json = {"workload": a.workload, "grid": list(grid), "odf": odf, "variant": a.variant, "launch": a.launch,
                "graph": bool(a.graph), "exchange": a.exchange, "overlap": bool(a.overlap), "n_gpus": n,
                "l2": "inputs larger than L2 (no flush needed)" if grid[0] * grid[1] * grid[2] * 16 / n > L2_BYTES
                else "inputs smaller than L2",
                "init": f"hash-random [0,1), seed {SEED}, Dirichlet 1.0"}

    if a.impl == "reference":
        if rank != 0:
            return
        return reference_arm(a, grid, cfg_json)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2202_11819_b200 as j3d
    from paper_2202_11819_b200 import dist as jdist

    if world > 1:
        ctx = jdist.create(grid, odf=odf, variant=a.variant, launch=a.launch, graph=bool(a.graph),
                           exchange=a.exchange, overlap=bool(a.overlap))
    else:
        ctx = j3d.Jacobi3D(grid, odf=odf, variant=a.variant, launch=a.launch, graph=bool(a.graph),
                           exchange=a.exchange, device=local)
    lups_step = grid[0] * grid[1] * grid[2]
    ctx.init("hash", seed=SEED)
    ctx.iterate(a.warmup)
    ctx.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.profile_enable(True)
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    reps = []
    for _ in range(max(1, a.repeats)):
        # CUDA events on the library's stream around exactly K steps (jacobi3d_time:
        # stream sync + barrier over ranks before the start event)
        ms_r = ctx.time(0, a.steps)
        t = torch.tensor([ms_r], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
        reps.append(float(t.item()))
    clocks = clk.stop()
    prof_ms, prof_n, prof_bytes = ctx.profile_read()
    ctx.profile_enable(False)
    st = ctx.stats()
    launches = st["kernel_launches"] // len(reps)  # per timed region of K steps
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = statistics.mean(reps)
    value = lups_step * a.steps / (ms * a.steps * 1e-3) / 1e9
    repeats = {"n": len(reps), "ms_per_step": [round(x, 4) for x in reps], "mean_ms": round(ms, 4),
               "min_ms": round(min(reps), 4), "value_mean": round(value, 3),
               "value_best": round(lups_step / (min(reps) * 1e-3) / 1e9, 3),
               "what": "value = mean over repeats of the max-over-ranks ms/step of K timed steps"}

    peak, peak_src = load_peaks()
    roof = None
    if prof_n > 0:
        avg_ms = prof_ms / prof_n
        achieved = (prof_bytes / prof_n) / (avg_ms * 1e-3) / 1e9
        if a.launch == "per_block":
            # per-block launches run concurrently on their own streams: their
            # event times overlap, so use all stencil bytes over the step time
            achieved = prof_bytes / (ms * a.steps * len(reps) * 1e-3) / 1e9
        tr, tr_src = traffic_from_profiles(a.workload, a.launch, a.variant, st.get("tile_kind"), a.steps)
        roof = {"bound": "hbm", "kernel": "stencil_tma_kernel", "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": tr["traffic_bytes_per_launch"] if tr else None, "traffic_source": tr_src,
                "tile_kind": st.get("tile_kind"),
                "alg_bytes_per_launch": prof_bytes / prof_n, "avg_launch_ms": avg_ms,
                "share_of_step": round(prof_ms / (ms * a.steps * len(reps)), 4), "peak_source": peak_src,
                "method": ("stencil bytes in the timed region / step time (per-block launches overlap)"
                           if a.launch == "per_block" else
                           "algorithmic bytes per launch / mean CUDA-event launch time")}

    e2e = None
    if not a.no_e2e:
        e2e = e2e_run(ctx, grid, a, world, rank)

    halo = None
    if world > 1:
        ctx.set_skip_exchange(True)
        ms_skip = ctx.time(3, max(10, a.steps // 4))
        ctx.set_skip_exchange(False)
        t2 = torch.tensor([ms_skip], dtype=torch.float64, device="cuda")
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        halo = {"exposed_halo_ms_per_iter": round(ms - float(t2.item()), 4),
                "ms_per_iter_exchange_elided": round(float(t2.item()), 4)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:  # the oracle baseline: rank 0 at N=1 only
        cpu = cpu_baseline(grid)

    ctx.close()
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GLUPS", "n_gpus": n, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling":
                "weak" if wl["kind"] == "weak" else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": cfg_json,
                "hbm_gbs_per_gpu": round(value / n * BYTES_PER_LUP, 1),
                "hbm_frac_per_gpu": round(value / n * BYTES_PER_LUP / peak, 4),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
                "repeats": repeats}
        if halo:
            line["halo"] = halo
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_run(ctx, grid, a, world, rank):
    """Same metric end to end through the C ABI with HOST buffers: upload of
    the initial field from pinned host memory (jacobi3d_set_block), K steps,
    device->host read of the final residual (the metric a solver monitors)
    and download of the final field (jacobi3d_get_block)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    ex = ctx.extent
    blocks = [b for b in range(ctx.n_blocks) if ctx.block_info(b)[2] == ctx.cfg.rank]
    nb = ex[0] * ex[1] * ex[2]
    # every rank on this node pins its whole field: only if it fits comfortably in host RAM
    need = 8 * nb * len(blocks) * int(os.environ.get("LOCAL_WORLD_SIZE", world))
    avail = 0
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    ok = torch.tensor([1.0 if need <= 0.45 * avail else 0.0], device="cuda")
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() < 1.0:
        return {"value": None, "unit": "GLUPS", "skipped": f"pinned host copies of the field need {need/1e9:.0f} GB, "
                f"MemAvailable {avail/1e9:.0f} GB on this node"}
    host = torch.empty(nb * len(blocks), dtype=torch.float64, pin_memory=True)
    hp = host.data_ptr()
    # synthetic initial field on the host (uniform [0,1), not timed)
    host.uniform_(0.0, 1.0, generator=torch.Generator().manual_seed(SEED + rank))
    ctx.init("default")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, b in enumerate(blocks):
        ctx.set_block_ptr(b, hp + 8 * nb * i)
    ctx.refresh_halos()
    ctx.iterate(a.steps)
    res = ctx.residual()
    for i, b in enumerate(blocks):
        ctx.get_block_ptr(b, hp + 8 * nb * i)
    ctx.synchronize()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el = float(t.item())
    lups = grid[0] * grid[1] * grid[2] * a.steps
    bytes_field = 8 * nb * len(blocks)
    del host
    return {"value": round(lups / el / 1e9, 3), "unit": "GLUPS", "seconds": round(el, 4),
            "h2d_bytes_per_step": bytes_field / a.steps, "d2h_bytes_per_step": bytes_field / a.steps + 8,
            "what": "H2D initial field (pinned) + K iterations + residual read + D2H final field, "
                    "wall clock, max over ranks", "last_residual": res}


def reference_arm(a, grid, cfg_json):
    """--impl reference: the CPU oracle as it stands, on the host cores; each
    step is one full oracle sweep of a bounded x-y-full slab of the workload."""
    from oracle import core

    gx, gy, gz = grid
    slab = max(4, min(gz, 32))
    U = core.init(gx, gy, slab, core.INIT_HASH, seed=SEED)
    V = U.copy()
    for _ in range(a.warmup):
        core.sweep_owned_timing(U, V)
        U, V = V, U
    t0 = time.perf_counter()
    for _ in range(a.steps):
        core.sweep_owned_timing(U, V)
        U, V = V, U
    el = time.perf_counter() - t0
    lups = gx * gy * slab * a.steps
    value = lups / el / 1e9
    sample = f"each step = one oracle sweep of a {gx}x{gy}x{slab} slab of the {gx}x{gy}x{gz} workload"
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GLUPS", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(el / a.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg_json,
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 4), "unit": "GLUPS", "cores": core.threads(), "kind": "oracle",
                             "sample": sample, **host_cpu()},
            "e2e": {"value": round(value, 4), "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
