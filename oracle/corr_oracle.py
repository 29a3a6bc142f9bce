"""Float64 restatement of the per-edge correlation lookup (Eq. 4).

TEST INFRASTRUCTURE ONLY.  PARITY UNPINNED by the reference: the reference
package has no correlation code or test (SPEC.md:14 puts Eq. 4 out of scope),
so this oracle *defines* the conventions and is pinned only by its own
known-answer tests (tests/test_corr_oracle.py):

  C(e, l, c, a, b) = < g[ii[e], c], f_l[jj[e]]( P'_l(e, c) + (b - r, a - r) ) >

* g: patch features (patches, p*p, C); f_l: frame features (frames, H_l, W_l, C)
  channels-last; level 1 is the 4x4 average pool of level 0 (DPVO-style pyramid);
* P'_l = coords / 4**l, coords given at level-0 feature resolution;
* bilinear sampling with out-of-bounds taps = 0, evaluated (exactly, since the
  dot product is linear) as the bilinear blend of integer-tap dot products
  over the (2r+2)^2 grid anchored at floor(P') - r;
* output (E, L, p*p, 2r+1, 2r+1).
"""

from __future__ import annotations

import numpy as np


def avg_pool4(fmap):
    """(F, H, W, C) -> (F, H//4, W//4, C) mean over 4x4 blocks."""
    f, h, w, c = fmap.shape
    h4, w4 = h // 4, w // 4
    x = np.asarray(fmap, dtype=np.float64)[:, :h4 * 4, :w4 * 4, :]
    return x.reshape(f, h4, 4, w4, 4, c).mean(axis=(2, 4))


def corr(gmap, fmaps, coords, ii, jj, radius=3):
    g = np.asarray(gmap, dtype=np.float64)
    coords = np.asarray(coords, dtype=np.float64)
    ii = np.asarray(ii, dtype=np.int64)
    jj = np.asarray(jj, dtype=np.int64)
    E, m = coords.shape[:2]
    D, O = 2 * radius + 2, 2 * radius + 1
    out = np.zeros((E, len(fmaps), m, O, O))
    for lvl, fm in enumerate(fmaps):
        f = np.asarray(fm, dtype=np.float64)
        _, H, W, _ = f.shape
        xy = coords * (0.25 ** lvl)
        finite = np.all(np.isfinite(xy) & (np.abs(xy) < 1e7), axis=-1)
        xy = np.where(finite[..., None], xy, -1e9)
        x0 = np.floor(xy[..., 0]).astype(np.int64)
        y0 = np.floor(xy[..., 1]).astype(np.int64)
        dx = np.where(finite, xy[..., 0] - x0, 0.0)
        dy = np.where(finite, xy[..., 1] - y0, 0.0)
        S = np.zeros((E, m, D, D))
        for a in range(D):
            for b in range(D):
                py = y0 - radius + a
                px = x0 - radius + b
                inb = (py >= 0) & (py < H) & (px >= 0) & (px < W)
                pyc = np.clip(py, 0, H - 1)
                pxc = np.clip(px, 0, W - 1)
                taps = f[jj[:, None], pyc, pxc]                  # (E, m, C)
                dots = np.einsum("emc,emc->em", taps, g[ii])
                S[:, :, a, b] = np.where(inb, dots, 0.0)
        wx = dx[..., None, None]
        wy = dy[..., None, None]
        out[:, lvl] = ((1 - wy) * ((1 - wx) * S[:, :, :-1, :-1] + wx * S[:, :, :-1, 1:])
                       + wy * ((1 - wx) * S[:, :, 1:, :-1] + wx * S[:, :, 1:, 1:]))
    return out
