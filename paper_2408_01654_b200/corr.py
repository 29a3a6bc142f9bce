"""Per-edge correlation lookup (K1) — the op the reference leaves out.

PAPER.md:158-164 (Eq. 4): for edge (i, k, j) with reprojected patch P'
(K2's pixels, scaled to feature resolution), every patch cell's feature g is
dotted with the bilinearly sampled frame features f_j on a 7x7 grid around
P', at two pyramid levels.  Computed on the fly by ``dpv_corr`` (the dense
correlation volume is never materialised).  Conventions are fixed by the
oracle (oracle/corr_oracle.py; parity is unpinned by the reference, which has
no correlation code — SPEC.md:14).

Layouts (channels-last): gmap (patches, 9, C); fmap (frames, H, W, C);
coords (E, 9, 2) float64 at level-0 feature resolution; ii/jj int32.
Output (E, levels, 9, 2r+1, 2r+1) float32.
"""

from __future__ import annotations

import torch

from . import _lib

_DT = {torch.float32: 0, torch.bfloat16: 1}


def pyramid(fmap: torch.Tensor):
    """[level0, level1] with level1 the 4x4 average pool (DPVO's pyramid), on the device."""
    f, h, w, c = fmap.shape
    out = torch.empty((f, h // 4, w // 4, c), dtype=fmap.dtype, device=fmap.device)
    _lib.check(_lib.lib().dpv_avg_pool4(_lib.ptr(fmap.contiguous()), f, h, w, c, _DT[fmap.dtype],
                                        _lib.ptr(out), _lib.stream_ptr()), "avg_pool4")
    return [fmap, out]


def corr(gmap: torch.Tensor, fmaps, coords: torch.Tensor, ii: torch.Tensor, jj: torch.Tensor,
         radius: int = 3, out: torch.Tensor | None = None,
         items_per_cta: int = 0) -> torch.Tensor:
    """K1 for every edge at every level of ``fmaps`` (``dpv_corr_ex2``).

    items_per_cta = 0 runs one persistent CTA per SM (fastest alone); > 0
    runs short-lived CTAs of that many (edge, level) items, for a lookup on
    a low-priority stream beside higher-priority work (bench.py runs it
    beside the BA solve with 32): the block scheduler then gives SMs back to
    the other stream at CTA granularity.  Results are identical."""
    levels = len(fmaps)
    if levels not in (1, 2):
        raise ValueError("1 or 2 pyramid levels")
    if gmap.dtype not in _DT or any(f.dtype != gmap.dtype for f in fmaps):
        raise TypeError("features must all be float32 or all bfloat16")
    E = int(coords.shape[0])
    C = int(gmap.shape[-1])
    O = 2 * radius + 1
    if out is None:
        out = torch.empty((E, levels, 9, O, O), dtype=torch.float32, device="cuda")
    f0 = fmaps[0].contiguous()
    f1 = fmaps[1].contiguous() if levels == 2 else None
    g = gmap.contiguous()
    _lib.check(_lib.lib().dpv_corr_ex2(
        _lib.ptr(g), int(g.shape[0]), _lib.ptr(f0), _lib.ptr(f1), int(f0.shape[0]),
        _lib.ptr(coords.to(torch.float64).contiguous()), _lib.ptr(ii.to(torch.int32).contiguous()),
        _lib.ptr(jj.to(torch.int32).contiguous()), E, C, f0.shape[1], f0.shape[2],
        f1.shape[1] if f1 is not None else 0, f1.shape[2] if f1 is not None else 0, levels,
        radius, _DT[gmap.dtype], int(items_per_cta), _lib.ptr(out), _lib.stream_ptr()), "corr")
    return out
