"""The bench.py JSON contract: the reference arm on CPU (runs here) and the
device arm on the GPU -- every key the driver and the judge read."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "cpu_baseline"}


def run_bench(args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    import oracle as O
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    d = run_bench(["--impl", "reference", "--scale", "12", "--steps", "1", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "iters/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_device_arm_contract():
    d = run_bench(["--scale", "16", "--steps", "2", "--warmup", "3", "--no-extras",
                   "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "iters/s" and d["dtype"] == "f32"
    assert d["gpu_launches"] > 0
    rl = d["roofline"]
    assert rl["bound"] == "hbm" and rl["unit"] == "GB/s" and rl["peak"] > 0
    assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-9
    assert rl["traffic"] is None  # the committed capture is for scale 24 only
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 4 * (1 << 16)
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)


def test_reference_arm_under_torchrun_prints_once():
    """N > 1 as the driver launches it: rank 0 alone runs the reference arm and
    prints one line; the other ranks exit 0 without work."""
    import socket
    import oracle as O
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), "bench.py", "--impl", "reference",
                        "--gpus", "2", "--scale", "12", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0


def test_reference_arm_default_is_the_device_arms_config():
    """`bench.py --impl reference` exactly as the driver runs it (no --scale):
    the same matrix as the device arm's N = 1 line, R-MAT scale 24 (C2)."""
    import oracle as O
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    d = run_bench(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=900)
    assert d["config"]["scale"] == 24 and d["config"]["n"] == 1 << 24
    assert d["value"] > 0 and d["impl"] == "reference"
