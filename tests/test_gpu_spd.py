"""GPU parity of the sparse band+border SPD solver (spd.cu) through the
C-ABI ``dpv_block_sparse_solve`` (the block-sparse backend,
block_cholesky.py:48-111 + BlockCholeskyFactor.solve 31-45).

Random SPD block matrices on patch-graph-like patterns (a band of odometry
couplings plus long-range loop-closure couplings) are solved on the
device and compared with ``numpy.linalg.solve`` on the dense matrix.
Tolerance: max |x - x_ref| <= 1e-9 * max |x_ref| (float64, well-conditioned).
The chain count of the nested-dissection split is forced through
DPV_SPD_CHAINS to cover 1, 2 and 3 concurrent chains.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_01654_b200 import block_cholesky  # noqa: E402
from paper_2408_01654_b200.errors import SingularSystem  # noqa: E402


def pattern(n, band, loops, rng):
    keys = set()
    for a in range(n):
        for b in range(a, min(n, a + band + 1)):
            keys.add((a, b))
    for _ in range(loops):
        old = int(rng.integers(0, max(1, n // 4)))
        recent = int(rng.integers(3 * n // 4, n))
        for o in range(max(0, old - band // 2), min(n, old + band // 2 + 1)):
            a, b = min(o, recent), max(o, recent)
            keys.add((a, b))
    return np.array(sorted(keys), dtype=np.int64)


def spd_blocks(keys, n, rng):
    blocks = rng.normal(size=(len(keys), 6, 6))
    dense = np.zeros((6 * n, 6 * n))
    for (a, b), blk in zip(keys, blocks):
        if a == b:
            blk[:] = 0.5 * (blk + blk.T)
        dense[6 * a:6 * a + 6, 6 * b:6 * b + 6] = blk
        dense[6 * b:6 * b + 6, 6 * a:6 * a + 6] = blk.T
    shift = np.abs(dense).sum(axis=1) + 1.0
    for (a, b), blk in zip(keys, blocks):
        if a == b:
            blk[np.diag_indices(6)] += shift[6 * a:6 * a + 6]
    dense[np.diag_indices(6 * n)] += shift
    return blocks, dense


def solve(keys, blocks, n, rhs):
    fac = block_cholesky.block_cholesky(keys, blocks, n)
    return fac.solve(rhs.reshape(n, 6)).reshape(-1)


@pytest.mark.parametrize("n,band,loops,chains", [
    (1, 0, 0, 0), (2, 1, 0, 0), (11, 2, 0, 0), (30, 30, 0, 0), (64, 3, 4, 0),
    (300, 13, 0, 1), (300, 13, 0, 2), (300, 13, 0, 3),
    (600, 26, 10, 0), (600, 26, 10, 1), (600, 26, 10, 2), (900, 20, 15, 3),
])
def test_block_sparse_solve_matches_dense(n, band, loops, chains, monkeypatch):
    if chains:
        monkeypatch.setenv("DPV_SPD_CHAINS", str(chains))
    else:
        monkeypatch.delenv("DPV_SPD_CHAINS", raising=False)
    rng = np.random.default_rng(n * 1000 + band * 10 + chains)
    keys = pattern(n, band, loops, rng)
    blocks, dense = spd_blocks(keys, n, rng)
    rhs = rng.normal(size=6 * n)
    x = solve(keys, blocks, n, rhs)
    ref = np.linalg.solve(dense, rhs)
    err = np.abs(x - ref).max()
    assert err <= 1e-9 * np.abs(ref).max(), err


def test_block_sparse_solve_is_deterministic():
    rng = np.random.default_rng(7)
    n = 500
    keys = pattern(n, 26, 8, rng)
    blocks, _ = spd_blocks(keys, n, rng)
    rhs = rng.normal(size=6 * n)
    a = solve(keys, blocks, n, rhs)
    b = solve(keys, blocks, n, rhs)
    assert np.array_equal(a, b)


def test_block_sparse_singular():
    rng = np.random.default_rng(3)
    n = 200
    keys = pattern(n, 13, 3, rng)
    blocks, _ = spd_blocks(keys, n, rng)
    diag = np.nonzero(keys[:, 0] == keys[:, 1])[0]
    blocks[diag[150]] = -np.eye(6)
    with pytest.raises(SingularSystem):
        block_cholesky.block_cholesky(keys, blocks, n)
    with pytest.raises(SingularSystem):      # missing diagonal block
        block_cholesky.block_cholesky(keys[keys[:, 0] != 5], blocks[keys[:, 0] != 5], n)


def test_long_chain_residual():
    """A cfg4-length band (4400 poses, ~413 band tiles: one co-resident
    substitution CTA per tile) solved through the block-sparse C-ABI; checked
    by the block residual ||S x - b|| (the dense matrix would take 5 GB)."""
    rng = np.random.default_rng(44)
    n, band = 4400, 13
    keys = pattern(n, band, 3, rng)
    blocks = rng.normal(size=(len(keys), 6, 6)) * 0.1
    diag = keys[:, 0] == keys[:, 1]
    blocks[diag] = 0.5 * (blocks[diag] + blocks[diag].transpose(0, 2, 1))
    # diagonal dominance per row from the off-diagonal block magnitudes
    rowsum = np.zeros(6 * n)
    for (a, b), blk in zip(keys[~diag], blocks[~diag]):
        rowsum[6 * a:6 * a + 6] += np.abs(blk).sum(axis=1)
        rowsum[6 * b:6 * b + 6] += np.abs(blk).sum(axis=0)
    for idx in np.nonzero(diag)[0]:
        a = keys[idx, 0]
        blocks[idx][np.diag_indices(6)] += rowsum[6 * a:6 * a + 6] + np.abs(blocks[idx]).sum(1) + 1
    rhs = rng.normal(size=6 * n)
    x = solve(keys, blocks, n, rhs)
    sx = np.zeros(6 * n)
    for (a, b), blk in zip(keys, blocks):
        sx[6 * a:6 * a + 6] += blk @ x[6 * b:6 * b + 6]
        if a != b:
            sx[6 * b:6 * b + 6] += blk.T @ x[6 * a:6 * a + 6]
    assert np.abs(sx - rhs).max() <= 1e-9 * np.abs(rhs).max()
