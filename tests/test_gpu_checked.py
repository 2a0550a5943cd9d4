"""The -DKMD_CHECKS build of libkmd (device-side bounds assertions on every
shared-memory index of the pipelined kernels, kmd_common.cuh KMD_CHECK) runs
one small case of every kernel family and compares each with the oracle
(scripts/sanitize_cases.py).  This stands in for compute-sanitizer, which is
closed on this run's GPU pool; a violated check traps, so the subprocess
fails."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_every_kernel_family():
    from paper_2202_05977_b200 import _build
    lib = _build.build(checked=True)
    env = dict(os.environ, KMD_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitize cases done" in r.stdout, out[-4000:]
    assert "KMD_CHECK failed" not in out


def test_checked_build_is_deterministic_under_scheduling_jitter(tmp_path):
    # KMD_DEBUG = seed makes every role of the checked TMA kernel sleep
    # pseudo-random 0-2 us at its protocol points (kmd_common.cuh KMD_JITTER):
    # the warps interleave differently, and a missing wait or an early slot
    # release would change the output.  Every seed must reproduce the
    # unperturbed run bit for bit.
    import numpy as np
    from paper_2202_05977_b200 import _build
    lib = _build.build(checked=True)
    outs = {}
    for seed in (0, 1, 2, 3):
        d = tmp_path / f"s{seed}"
        env = dict(os.environ, KMD_LIB=lib, KMD_DEBUG=str(seed))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "jitter_cases.py"), str(d)], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and "jitter cases done" in r.stdout, (r.stdout + r.stderr)[-4000:]
        outs[seed] = {n: np.load(d / f"{n}.npy") for n in ("m6", "m3", "mr")}
    for seed in (1, 2, 3):
        for n in ("m6", "m3", "mr"):
            assert np.array_equal(outs[seed][n], outs[0][n]), (seed, n)
