"""GPU parity of the correlation kernel (K1) against the float64 oracle.

Tolerance: float32 accumulation over C=128 channels of unit-variance / sqrt(C)
features -> |err| <= 2e-5 (fp32 features); bf16 features are compared with
the oracle evaluated on the same bf16 values -> |err| <= 2e-4 (bf16 output of
the level-1 pool is rounded once more).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import corr_oracle  # noqa: E402
from paper_2408_01654_b200 import corr  # noqa: E402


def make(rng, E=300, C=128, F=4, H=30, W=40, P=50, spread=1.0):
    g = (rng.normal(size=(P, 9, C)) / np.sqrt(C)).astype(np.float32)
    f = (rng.normal(size=(F, H, W, C)) / np.sqrt(C)).astype(np.float32)
    base = rng.uniform(-3, [W + 3, H + 3], size=(E, 1, 2))
    offs = np.stack(np.meshgrid(np.arange(3) - 1.0, np.arange(3) - 1.0), -1).reshape(1, 9, 2)
    coords = base + spread * offs * rng.uniform(0.1, 0.3) + rng.normal(0, 0.05, (E, 9, 2))
    ii = rng.integers(0, P, E).astype(np.int32)
    jj = rng.integers(0, F, E).astype(np.int32)
    return g, f, coords, ii, jj


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_corr_matches_oracle(dtype):
    rng = np.random.default_rng(0)
    g, f, coords, ii, jj = make(rng)
    coords[0] = np.nan
    coords[1] += 500.0                       # fully out of bounds
    coords[2, :, 0] = np.linspace(-1, 60, 9)  # cells spread wider than the staged window
    gd = torch.as_tensor(g, device="cuda").to(dtype)
    fd = torch.as_tensor(f, device="cuda").to(dtype)
    pyr = corr.pyramid(fd)
    out = corr.corr(gd, pyr, torch.as_tensor(coords, device="cuda"),
                    torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda"))
    g64 = gd.double().cpu().numpy()
    f64 = fd.double().cpu().numpy()
    f1 = pyr[1].double().cpu().numpy()
    ref = corr_oracle.corr(g64, [f64, f1], coords, ii, jj)
    tol = 2e-5 if dtype == torch.float32 else 2e-4
    err = np.abs(out.cpu().numpy() - ref).max()
    assert err < tol, err
    assert np.all(out[:2].cpu().numpy() == 0)
    if dtype == torch.float32:
        assert np.allclose(pyr[1].cpu().numpy(), corr_oracle.avg_pool4(f), atol=1e-6)


@pytest.mark.parametrize("E,C", [(3000, 128), (2000, 64), (1500, 256)])
def test_corr_bf16_tensor_core_pipeline(E, C):
    """Several items per CTA (double-buffered staging) and every channel
    count with a tensor-core instantiation, against the oracle on the same
    bf16 values."""
    rng = np.random.default_rng(E + C)
    g, f, coords, ii, jj = make(rng, E=E, C=C, F=6, H=24, W=32, P=80)
    coords[5::97, :, 1] = np.linspace(0, 40, 9)      # some wide windows (fallback)
    gd = torch.as_tensor(g, device="cuda").to(torch.bfloat16)
    fd = torch.as_tensor(f, device="cuda").to(torch.bfloat16)
    pyr = corr.pyramid(fd)
    out = corr.corr(gd, pyr, torch.as_tensor(coords, device="cuda"),
                    torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda"))
    ref = corr_oracle.corr(gd.double().cpu().numpy(),
                           [fd.double().cpu().numpy(), pyr[1].double().cpu().numpy()],
                           coords, ii, jj)
    err = np.abs(out.cpu().numpy() - ref).max()
    assert err < 2e-4 * np.sqrt(C / 128), err


def test_corr_on_reprojected_patches():
    """K2 -> K1: correlation at the BA problem's reprojections peaks at the
    center when the features of frame j are those sampled from the truth."""
    rng = np.random.default_rng(1)
    C, H, W = 64, 40, 52
    f = (rng.normal(size=(1, H, W, C)) / 8).astype(np.float32)
    coords = rng.uniform(5, 30, size=(40, 1, 2)).round() + np.stack(
        np.meshgrid(np.arange(3.0), np.arange(3.0)), -1).reshape(1, 9, 2)
    g = np.stack([[f[0, int(y), int(x)] for x, y in c] for c in coords]).astype(np.float32)
    out = corr.corr(torch.as_tensor(g, device="cuda"), [torch.as_tensor(f, device="cuda")],
                    torch.as_tensor(coords, device="cuda"),
                    torch.arange(40, dtype=torch.int32, device="cuda"),
                    torch.zeros(40, dtype=torch.int32, device="cuda"))
    flat = out[:, 0].reshape(40, 9, 49).argmax(-1).cpu().numpy()
    assert np.all(flat == 24)


def bench_shape_case(rng, E, H, W, F=24, P=4000, C=128):
    """Edges at the bench feature shapes (cfg3 1/4-res 120x160, cfg4 KITTI
    92x306), patch spreads as in a 3x3 patch reprojected at 1/4 resolution."""
    g = (rng.normal(size=(P, 9, C)) / np.sqrt(C)).astype(np.float32)
    f = (rng.normal(size=(F, H, W, C)) / np.sqrt(C)).astype(np.float32)
    base = rng.uniform(-2, [W + 2, H + 2], size=(E, 1, 2))
    offs = np.stack(np.meshgrid(np.arange(3) - 1.0, np.arange(3) - 1.0), -1).reshape(1, 9, 2)
    coords = base + 0.25 * offs * rng.uniform(0.7, 1.4, size=(E, 1, 1))
    ii = rng.integers(0, P, E).astype(np.int32)
    jj = np.sort(rng.integers(0, F, E)).astype(np.int32)     # grouped by target frame
    return g, f, coords, ii, jj


@pytest.mark.parametrize("H,W", [(120, 160), (92, 306)])
def test_corr_bench_shapes(H, W):
    """Full bench-size launch (48k edges, both levels, C=128 bf16) checked on
    a seeded sample of 1500 edges: (1) against the oracle on the same bf16
    values (kernel arithmetic: |err| <= 2e-4), (2) against the oracle on the
    ORIGINAL fp32 features -- the end-to-end error of storing features in
    bf16, stated tolerance |err| <= 4e-3 absolute and RMS error <= 1% of
    the output RMS (outputs ~ N(0, 0.09^2))."""
    rng = np.random.default_rng(H * W)
    E = 48_000
    g, f, coords, ii, jj = bench_shape_case(rng, E, H, W)
    gd = torch.as_tensor(g, device="cuda").bfloat16()
    fd = torch.as_tensor(f, device="cuda").bfloat16()
    pyr = corr.pyramid(fd)
    out = corr.corr(gd, pyr, torch.as_tensor(coords, device="cuda"),
                    torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda"))
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    sel = np.sort(rng.choice(E, 1500, replace=False))
    got = out.cpu().numpy()[sel]
    ref_b = corr_oracle.corr(gd.double().cpu().numpy(),
                             [fd.double().cpu().numpy(), pyr[1].double().cpu().numpy()],
                             coords[sel], ii[sel], jj[sel])
    assert np.abs(got - ref_b).max() < 2e-4
    ref_f = corr_oracle.corr(g, [f, corr_oracle.avg_pool4(f)], coords[sel], ii[sel], jj[sel])
    err = got - ref_f
    assert np.abs(err).max() < 4e-3, np.abs(err).max()
    assert np.sqrt((err ** 2).mean()) < 0.01 * np.sqrt((ref_f ** 2).mean())


def test_corr_single_level_and_odd_counts():
    """One pyramid level, edge counts that do not fill the last round of
    items, C=64 (12-stage ring)."""
    rng = np.random.default_rng(7)
    for E in (1, 149, 1001):
        g, f, coords, ii, jj = make(rng, E=E, C=64, F=3, H=28, W=36, P=40)
        gd = torch.as_tensor(g, device="cuda").bfloat16()
        fd = torch.as_tensor(f, device="cuda").bfloat16()
        out = corr.corr(gd, [fd], torch.as_tensor(coords, device="cuda"),
                        torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda"))
        ref = corr_oracle.corr(gd.double().cpu().numpy(), [fd.double().cpu().numpy()],
                               coords, ii, jj)
        assert out.shape == (E, 1, 9, 7, 7)
        assert np.abs(out.cpu().numpy() - ref).max() < 2e-4


@pytest.mark.parametrize("items", [1, 7, 48, 10_000])
def test_corr_items_per_cta_identical(items):
    """Short-lived CTAs (items_per_cta > 0: the lookup beside the solve on a
    low-priority stream) compute exactly the persistent kernel's outputs,
    including item counts that leave ragged last chunks."""
    rng = np.random.default_rng(11 + items)
    E = 5_003
    g, f, coords, ii, jj = bench_shape_case(rng, E, 120, 160, F=6, P=500)
    gd = torch.as_tensor(g, device="cuda").bfloat16()
    pyr = corr.pyramid(torch.as_tensor(f, device="cuda").bfloat16())
    args = (gd, pyr, torch.as_tensor(coords, device="cuda"), torch.as_tensor(ii, device="cuda"),
            torch.as_tensor(jj, device="cuda"))
    ref = corr.corr(*args)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        got = corr.corr(*args, items_per_cta=items)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    with pytest.raises(Exception):
        corr.corr(*args, items_per_cta=-1)
