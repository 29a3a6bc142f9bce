"""CPU checks of the C-ABI boundary: the in-tree library loads and exports
every entry point include/dpvslam_b200.h declares (no compute calls)."""

import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dpvslam_b200.h")).read()
    return sorted(set(re.findall(r"\b(dpv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("dpv_problem_create", "dpv_assemble", "dpv_solve", "dpv_lm_solve",
                 "dpv_reproject_grid", "dpv_objective", "dpv_corr", "dpv_apply_step"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2408_01654_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2408_01654_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    loaded = _lib.load(require_gpu=False)
    assert loaded.dpv_abi_version() == 1
    assert loaded.dpv_last_error() == b""


def test_no_gpu_means_loud_failure():
    import torch
    from paper_2408_01654_b200 import _lib
    from paper_2408_01654_b200.errors import NativeUnavailable
    if torch.cuda.is_available():
        return
    try:
        _lib.lib()
    except NativeUnavailable:
        return
    raise AssertionError("the product path must not run without a GPU")
