"""The bench.py contract on CPU: the reference arm (the CPU oracle) prints one
JSON line with the keys the driver reads; argument validation."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                        "--warmup", "3", "--workload", "small64_odf8"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GLUPS" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "small64_odf8"


def test_warmup_must_be_at_least_three():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=120)
    assert p.returncode != 0


def test_workload_launch_defaults_in_config():
    """The reference arm reports the same config as the GPU arm, including the
    launch mode each workload defaults to (persistent for the small and
    fine-grained grids, batched for the 1536^3 ones and for non-direct variants)."""
    def cfg(*args):
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                            "--warmup", "3", *args], capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        return json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])["config"]

    assert cfg("--workload", "small64_odf8")["launch"] == "batched"
    assert cfg("--workload", "small192_odf1", "--grid", "64,64,32")["launch"] == "persistent"
    assert cfg("--workload", "small192_odf1", "--grid", "64,64,32", "--variant", "unfused")["launch"] == "batched"
    assert cfg("--workload", "small192_odf1", "--grid", "64,64,32", "--launch", "per_block")["launch"] == "per_block"


def test_weak_scaling_grids_plan_to_fixed_per_gpu_work():
    """Weak scaling as the driver runs it (N = 1, 2, 4, 8, one rank per GPU):
    for every weak workload bench.py's global grid plans to the GPU grid
    weak_global assumes, each GPU owns exactly the per-GPU block split into ODF
    blocks, peer faces per GPU are 0/1/2/3 and the plan fits one
    B200's 180 GB of HBM."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2202_11819_b200 as j3d

    want_grid = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}
    for name, wl in bench.WORKLOADS.items():
        if wl["kind"] != "weak":
            continue
        for n, faces in ((1, 0), (2, 1), (4, 2), (8, 3)):
            g = bench.weak_global(wl["per_gpu"], n)
            info = j3d.plan(g, odf=wl["odf"], n_gpus=n, launch=wl.get("launch", "batched"))
            assert info["gpu_grid"] == want_grid[n], (name, n, info)
            per_gpu = tuple(b * k for b, k in zip(info["blk_ext"], info["blk_grid"]))
            assert per_gpu == tuple(wl["per_gpu"]), (name, n, info)
            assert info["n_blocks"] == wl["odf"] * n
            if wl["odf"] == 1:
                assert info["peer_faces_max"] == faces, (name, n, info)
            assert 0 < info["bytes_per_gpu"] < 180e9, (name, n, info["bytes_per_gpu"])


def test_traffic_only_from_a_matching_capture(tmp_path, monkeypatch):
    """roofline.traffic comes from a committed ncu capture only when it was taken from
    the same sources (build_sha256), workload, launch mode, variant, tile kind and --
    for the persistent launch -- iterations per launch; otherwise None and the reason."""
    import shutil

    sys.path.insert(0, ROOT)
    import bench

    sha = bench.build_sha256()
    assert sha == bench.build_sha256() and len(sha) == 64  # deterministic over the sources
    prof = tmp_path / "profiles"
    prof.mkdir()
    cap = {"workload": "weak1536_odf1", "launch": "batched", "variant": "direct", "tile_kind": 26,
           "iters_per_launch": 1, "build_sha256": sha, "traffic_bytes_per_launch": 5.9e10}
    (prof / "ncu_stencil_x.json").write_text(json.dumps(cap))
    # build_sha256 hashes ROOT's sources: give the temporary root the same ones
    for sub in ("paper_2202_11819_b200/csrc", "include"):
        shutil.copytree(os.path.join(ROOT, sub), tmp_path / sub)
    shutil.copy(os.path.join(ROOT, "paper_2202_11819_b200", "build.py"), tmp_path / "paper_2202_11819_b200")
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    d, src = bench.traffic_from_profiles("weak1536_odf1", "batched", "direct", 26, 20)
    assert d and d["traffic_bytes_per_launch"] == 5.9e10 and src == "ncu_stencil_x.json"
    assert bench.traffic_from_profiles("weak1536_odf1", "batched", "direct", 0, 20)[0] is None  # tile kind
    assert bench.traffic_from_profiles("weak1536_odf1", "persistent", "direct", 26, 20)[0] is None  # launch
    cap.update(launch="persistent", iters_per_launch=100)
    (prof / "ncu_stencil_x.json").write_text(json.dumps(cap))
    assert bench.traffic_from_profiles("weak1536_odf1", "persistent", "direct", 26, 100)[0] is not None
    assert bench.traffic_from_profiles("weak1536_odf1", "persistent", "direct", 26, 20)[0] is None  # iterations
    with open(tmp_path / "paper_2202_11819_b200" / "csrc" / "kernels.cu", "a") as f:
        f.write("// edited\n")
    d, why = bench.traffic_from_profiles("weak1536_odf1", "persistent", "direct", 26, 100)
    assert d is None and "build_sha256" in why  # a source edit invalidates the capture
