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
