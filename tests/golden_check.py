"""Comparison helpers for the config-scale golden files (make_golden_cfg.py)."""

import hashlib

import numpy as np


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a)).tobytes()).hexdigest()


def check(z, key, a, rel, abs_=0.0):
    a = np.asarray(a, dtype=np.float64)
    if "full_" + key in z:
        b = z["full_" + key]
        assert a.shape == b.shape, (key, a.shape, b.shape)
        scale = max(1.0, float(np.abs(b).max())) if b.size else 1.0
        err = float(np.abs(a - b).max()) if b.size else 0.0
        assert err <= abs_ + rel * scale, f"{key}: max err {err:.3e} (scale {scale:.3e})"
        return
    idx = z["smp_" + key + "_idx"]
    b = z["smp_" + key + "_val"]
    s = z["sum_" + key]
    scale = max(1.0, float(s[2]))
    err = float(np.abs(a[idx] - b).max())
    assert err <= abs_ + rel * scale, f"{key}: sampled max err {err:.3e} (scale {scale:.3e})"
    mine = np.array([a.sum(), np.abs(a).sum(), np.abs(a).max()])
    assert abs(mine[1] - s[1]) <= rel * s[1] + abs_ * a.size, (key, mine, s)
    assert abs(mine[0] - s[0]) <= rel * s[1] + abs_ * a.size, (key, mine, s)
    assert abs(mine[2] - s[2]) <= rel * scale + abs_, (key, mine, s)
