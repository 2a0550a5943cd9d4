"""bench.py's JSON contract on the GPU: one line with the driver's keys, a
roofline block, clocks, an e2e measurement through the C ABI with host
buffers, the kernel variant, and the CPU oracle baseline with a parity
number (small size, so the test stays fast)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_default_mode_json_contract():
    d = _run("--steps", "40", "--warmup", "3", "--height", "270", "--width", "480", "--e2e-steps", "3",
             "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 40 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and 0 < rf["frac"] < 1 and rf["peak"] > 1000
    assert "v3-tma-M6" in rf["kernel"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["parity"]["max_rel_err"] <= 1e-5
    assert d["gpu_launches"] == 40
    assert "workload" in d["config"]


@pytest.mark.parametrize("mode", ["mr", "bwd", "temporal"])
def test_next_row_modes_json(mode):
    d = _run("--mode", mode, "--steps", "16", "--warmup", "3", "--height", "272", "--width", "480")
    assert d["value"] > 0 and 0 < d["roofline"]["frac"] < 1 and "workload" in d["config"]


def test_bf16_mode_e2e_copies_bf16_inputs():
    H, W = 272, 480
    d = _run("--bf16", "--steps", "16", "--warmup", "3", "--height", str(H), "--width", str(W), "--e2e-steps", "3",
             "--no-cpu-baseline")
    e = d["e2e"]
    assert "host_bf16" in e["path"] and e["value"] > 0
    # radiance fp32 (3 planes) + importance and logits bf16 (6 + 6 planes)
    assert e["h2d_bytes_per_step"] == H * W * (3 * 4 + 12 * 2)
    assert e["d2h_bytes_per_step"] == H * W * 3 * 4
