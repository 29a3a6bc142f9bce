"""Float64 restatement of proximity loop-closure detection — TEST
INFRASTRUCTURE ONLY (the checker of ``dpv_proximity_detect``).

Follows pkg/src/patchslam/loop.py:51-85: the gate defaults to twice the
median inter-frame camera-centre spacing (resolve_threshold, loop.py:51-61);
a pair (old, recent) qualifies when recent - old >= min_temporal_gap and the
centre distance is below the gate; candidates are sorted by distance with
ties in insertion order (recent ascending, then old ascending; Python's sort
is stable).  Pinned against tests/golden/detect.npz (reference output).
"""

from __future__ import annotations

import numpy as np


def resolve_threshold(centers, distance_threshold=None):
    if distance_threshold is not None:
        return float(distance_threshold)
    centers = np.asarray(centers, dtype=float)
    if len(centers) < 2:
        return 0.0
    spacing = np.linalg.norm(np.diff(centers, axis=0), axis=1)
    return 2.0 * float(np.median(spacing))


def detect(centers, gap, threshold, newest=None):
    centers = np.asarray(centers, dtype=float)
    n = len(centers) if newest is None else newest + 1
    if n < gap + 1 or threshold <= 0:
        return []
    c = centers[:n]
    out = []
    for recent in range(gap, n):
        old = np.arange(0, recent - gap + 1)
        dist = np.linalg.norm(c[old] - c[recent], axis=1)
        hit = dist < threshold
        out.extend(zip(dist[hit], old[hit].tolist(), [recent] * int(hit.sum())))
    out.sort(key=lambda r: r[0])
    return [(int(o), int(r)) for _, o, r in out]
