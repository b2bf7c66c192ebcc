"""Frame-vs-ground-truth scores, plain numpy (SPEC metrics S:401-437).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the definition the CUDA
scores (libesi esi_frame_metrics) are checked against.

score_frame(recon, truth) -> (pearson, mse_norm): the Pearson correlation of the
frame's pixel values with the ground-truth log-intensity field, and the
mean squared error after per-image zero-mean unit-variance normalisation
(S:406).  Either image constant -> (nan, nan) ("missing").
"""
import numpy as np


def score_frame(recon, truth):
    x = np.asarray(recon, np.float64).ravel()
    y = np.asarray(truth, np.float64).ravel()
    if x.shape != y.shape:
        raise ValueError("GeometryMismatch")
    sx, sy = x.std(), y.std()
    if sx == 0.0 or sy == 0.0:
        return float("nan"), float("nan")
    zx = (x - x.mean()) / sx
    zy = (y - y.mean()) / sy
    return float(np.mean(zx * zy)), float(np.mean((zx - zy) ** 2))


def score_run(frames, truths):
    """Per-frame scores plus the summary of S:419 (mean / min over frames with a
    defined pearson, and how many were missing)."""
    sc = [score_frame(f, t) for f, t in zip(frames, truths)]
    p = np.array([s[0] for s in sc])
    ok = ~np.isnan(p)
    return sc, {"mean": float(p[ok].mean()) if ok.any() else float("nan"),
                "min": float(p[ok].min()) if ok.any() else float("nan"), "missing": int((~ok).sum())}
