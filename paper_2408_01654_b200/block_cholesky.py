"""Drop-in for patchslam.block_cholesky (block_cholesky.py:1-111).

``block_cholesky(keys, blocks, n)`` factors the SPD block matrix given by its
upper-triangle 6x6 block pattern, like the reference's right-looking block
factorisation — on the B200: the pattern is permuted into a band plus a thin
border (the reference keeps natural order and inserts fill dynamically; the
banded-plus-loop structure is the same observation, block_cholesky.py:1-8)
and factored by one dataflow kernel on the FP64 tensor cores (C-ABI
``dpv_block_sparse_solve``, spd.cu).  ``block_count`` is the exact
natural-order symbolic fill of the reference factorisation
(``dpv_block_fill_count``).  ``SingularSystem`` is raised for a missing
diagonal block or a non-positive-definite matrix, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C
import numpy as np

from . import _lib
from .errors import SingularSystem

BLOCK = 6


def _sparse_solve(keys, blocks_dev, n, rhs_dev):
    """x = S^-1 rhs on the device; raises SingularSystem if S is not SPD."""
    import torch
    x = torch.empty(BLOCK * n, dtype=torch.float64, device="cuda")
    status = torch.zeros(8, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().dpv_block_sparse_solve(
        keys.ctypes.data_as(C.c_void_p), len(keys), int(n), _lib.ptr(blocks_dev),
        _lib.ptr(rhs_dev), _lib.ptr(x), _lib.ptr(status), _lib.stream_ptr()),
        "block_cholesky")
    st = status.cpu().numpy()
    if st[0] != 0:
        raise SingularSystem(f"block {int(st[1]) // BLOCK} (permuted order) is not positive "
                             "definite")
    return x


@dataclass
class BlockCholeskyFactor:
    n: int
    block_count: int
    _keys: object = None        # (w, 2) int64 host pattern
    _blocks: object = None      # (w, 36) device copy of the blocks

    def solve(self, rhs):
        """Solve S x = rhs, rhs (n, 6) (block_cholesky.py:31-45), on the device."""
        import torch
        b = torch.as_tensor(np.ascontiguousarray(rhs, dtype=np.float64).reshape(-1),
                            device="cuda")
        x = _sparse_solve(self._keys, self._blocks, self.n, b)
        return x.reshape(self.n, BLOCK).cpu().numpy()


def block_cholesky(keys, blocks, n: int) -> BlockCholeskyFactor:
    import torch
    lib = _lib.lib()
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int64).reshape(-1, 2))
    n = int(n)
    present = np.zeros(n, dtype=bool)
    present[keys[keys[:, 0] == keys[:, 1], 0]] = True
    if not present.all():           # block_cholesky.py:73-76
        raise SingularSystem(f"missing diagonal block {int(np.argmin(present))}")
    count = C.c_int64()
    _lib.check(lib.dpv_block_fill_count(keys.ctypes.data_as(C.c_void_p), len(keys), n,
                                        C.byref(count)), "block_cholesky")
    blk = torch.as_tensor(np.ascontiguousarray(blocks, dtype=np.float64).reshape(-1, 36),
                          device="cuda")
    # factor once now so a non-SPD matrix raises here, as in the reference
    _sparse_solve(keys, blk, n, torch.zeros(BLOCK * n, dtype=torch.float64, device="cuda"))
    return BlockCholeskyFactor(n, int(count.value), keys, blk)
