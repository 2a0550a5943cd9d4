"""Parity helpers shared by the GPU tests (test infrastructure)."""
import numpy as np

# north_star: "max relative error <= 1e-5 in fp32" (BASELINE.json); DESIGN.md §5
REL_TOL = 1e-5


def rel_err(gpu: np.ndarray, ref: np.ndarray):
    """Max |gpu - ref| / |ref| over all elements (ref == 0 requires gpu == 0)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    zero = ref == 0
    if np.any(zero):
        assert np.all(gpu[zero] == 0), "oracle is exactly 0 but the GPU is not"
    d = np.abs(gpu - ref)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(zero, 0.0, d / np.abs(ref))
    i = int(np.argmax(rel))
    return float(rel.flat[i]), np.unravel_index(i, rel.shape), float(d.max())


def assert_parity(gpu, ref, tol=REL_TOL, what=""):
    assert np.all(np.isfinite(gpu)), f"{what}: non-finite GPU output"
    e, where, abs_max = rel_err(gpu, ref)
    assert e <= tol, f"{what}: max rel err {e:.3e} at {where} (max abs {abs_max:.3e}) > {tol}"
    return e
