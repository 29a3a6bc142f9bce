"""Known-answer tests pinning the correlation oracle (parity unpinned by the
reference, which has no correlation code: SPEC.md:14)."""

import numpy as np

from oracle.corr_oracle import avg_pool4, corr


def rand_inputs(rng, E=6, C=8, H=20, W=24, F=3, P=4):
    g = rng.normal(size=(P, 9, C))
    f = rng.normal(size=(F, H, W, C))
    ii = rng.integers(0, P, E)
    jj = rng.integers(0, F, E)
    return g, f, ii, jj


def test_integer_coords_equal_plain_dot():
    rng = np.random.default_rng(0)
    g, f, ii, jj = rand_inputs(rng)
    coords = np.tile(np.array([9.0, 7.0]), (6, 9, 1))
    out = corr(g, [f], coords, ii, jj)
    # Delta = (b - 3, a - 3); integer position -> exact tap
    for e in range(6):
        for c in range(9):
            for a in range(7):
                for b in range(7):
                    want = f[jj[e], 7 + a - 3, 9 + b - 3] @ g[ii[e], c]
                    assert abs(out[e, 0, c, a, b] - want) < 1e-12


def test_bilinear_equals_sampled_feature():
    rng = np.random.default_rng(1)
    g, f, ii, jj = rand_inputs(rng)
    coords = rng.uniform(4, 14, size=(6, 9, 2))
    out = corr(g, [f], coords, ii, jj)
    for e in range(6):
        for c in range(9):
            x, y = coords[e, c]
            a, b = 3, 3
            x0, y0 = int(np.floor(x)), int(np.floor(y))
            dx, dy = x - x0, y - y0
            samp = ((1 - dy) * (1 - dx) * f[jj[e], y0, x0] + (1 - dy) * dx * f[jj[e], y0, x0 + 1]
                    + dy * (1 - dx) * f[jj[e], y0 + 1, x0] + dy * dx * f[jj[e], y0 + 1, x0 + 1])
            assert abs(out[e, 0, c, a, b] - samp @ g[ii[e], c]) < 1e-12


def test_out_of_bounds_is_zero_and_nonfinite_safe():
    rng = np.random.default_rng(2)
    g, f, ii, jj = rand_inputs(rng)
    coords = np.full((6, 9, 2), -50.0)
    coords[0] = np.nan
    coords[1] = np.inf
    out = corr(g, [f], coords, ii, jj)
    assert np.all(out == 0)


def test_peak_at_true_position():
    rng = np.random.default_rng(3)
    C, H, W = 32, 24, 24
    f = rng.normal(size=(1, H, W, C))
    coords = np.stack(np.meshgrid(np.arange(3) + 10.0, np.arange(3) + 11.0), -1).reshape(1, 9, 2)
    g = np.stack([f[0, int(y), int(x)] for x, y in coords[0]])[None]
    out = corr(g, [f], coords, np.array([0]), np.array([0]))
    for c in range(9):
        assert np.argmax(out[0, 0, c]) == 3 * 7 + 3


def test_channel_linearity_and_pyramid():
    rng = np.random.default_rng(4)
    g, f, ii, jj = rand_inputs(rng, H=32, W=32)
    coords = rng.uniform(0, 31, size=(6, 9, 2))
    f1 = avg_pool4(f)
    assert f1.shape == (3, 8, 8, 8)
    assert np.allclose(f1[0, 1, 2], f[0, 4:8, 8:12].mean(axis=(0, 1)))
    a = corr(g, [f, f1], coords, ii, jj)
    b = corr(2.0 * g, [f, f1], coords, ii, jj)
    assert a.shape == (6, 2, 9, 7, 7)
    assert np.allclose(b, 2 * a)
