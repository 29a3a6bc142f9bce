"""Drop-in for patchslam.block_cholesky (block_cholesky.py:1-111).

``block_cholesky(keys, blocks, n)`` factors the SPD block matrix given by its
upper-triangle 6x6 block pattern.  The numeric factorisation runs on the B200
(dense FP64 Cholesky, trailing update on DMMA tensor cores, C-ABI
``dpv_cholesky_solve``); ``block_count`` is the exact natural-order symbolic
fill of the reference's right-looking block factorisation
(``dpv_block_fill_count``).  ``SingularSystem`` is raised for a missing
diagonal block or a non-positive-definite matrix, as in the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import SingularSystem

BLOCK = 6


@dataclass
class BlockCholeskyFactor:
    n: int
    block_count: int
    _matrix: object = None      # (6n, 6n) device copy of S (lower triangle used)

    def solve(self, rhs):
        """Solve S x = rhs, rhs (n, 6) (block_cholesky.py:31-45), on the device
        (factor + forward/backward substitution through dpv_cholesky_solve)."""
        import torch
        a = self._matrix.clone()
        b = torch.as_tensor(np.ascontiguousarray(rhs, dtype=np.float64).reshape(-1),
                            device="cuda").clone()
        status = torch.zeros(8, dtype=torch.int32, device="cuda")
        _lib.check(_lib.lib().dpv_cholesky_solve(_lib.ptr(a), _lib.ptr(b), a.shape[0],
                                                 _lib.ptr(status), _lib.stream_ptr()),
                   "BlockCholeskyFactor.solve")
        return b.reshape(self.n, BLOCK).cpu().numpy()


def dense_from_blocks(keys, blocks, n):
    full = np.zeros((BLOCK * n, BLOCK * n))
    for (a, b), blk in zip(np.asarray(keys).tolist(), blocks):
        full[6 * a:6 * a + 6, 6 * b:6 * b + 6] = blk
        if a != b:
            full[6 * b:6 * b + 6, 6 * a:6 * a + 6] = np.asarray(blk).T
    return full


def block_cholesky(keys, blocks, n: int) -> BlockCholeskyFactor:
    import torch
    lib = _lib.lib()
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int64).reshape(-1, 2))
    count = C.c_int64()
    _lib.check(lib.dpv_block_fill_count(keys.ctypes.data_as(C.c_void_p), len(keys), int(n),
                                        C.byref(count)), "block_cholesky")
    N = BLOCK * int(n)
    full = torch.as_tensor(dense_from_blocks(keys, blocks, n), device="cuda")
    a = full.clone()
    b = torch.zeros(N, dtype=torch.float64, device="cuda")
    status = torch.zeros(8, dtype=torch.int32, device="cuda")
    _lib.check(lib.dpv_cholesky_solve(_lib.ptr(a), _lib.ptr(b), N, _lib.ptr(status),
                                      _lib.stream_ptr()), "block_cholesky")
    st = status.cpu().numpy()
    if st[0] != 0:
        raise SingularSystem(f"diagonal block {int(st[1]) // BLOCK} is not positive definite")
    return BlockCholeskyFactor(int(n), int(count.value), full)
