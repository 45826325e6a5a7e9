"""Shared helpers for the GPU parity tests (no method arithmetic: comparisons only)."""
import numpy as np

TOL_BF16 = 2e-2     # BASELINE.json north_star: max-abs 2e-2 relative to logit scale (bf16)


def scale_of(ref):
    return max(1.0, float(np.max(np.abs(ref))))


def assert_close_scaled(got, ref, tol=TOL_BF16, what=""):
    s = scale_of(ref)
    err = float(np.max(np.abs(np.asarray(got, np.float64) - np.asarray(ref, np.float64))))
    assert err <= tol * s, f"{what}: max |diff| {err:.3e} > {tol} x scale {s:.3f}"
    return err / s


def rel_rms(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.sqrt(np.mean((got - ref) ** 2)) / max(1e-30, np.sqrt(np.mean(ref ** 2))))
