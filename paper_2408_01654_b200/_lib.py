"""ctypes binding of the C-ABI (include/dpvslam_b200.h).

This is the same binding a maintainer would add to the reference package
(INTEGRATION.md).  There is no CPU fallback: if the shared library or a CUDA
device is missing, every entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import NativeUnavailable, SingularSystem

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdpvslam_b200.so")

DPV_OK, DPV_SINGULAR, DPV_BAD_ARGS, DPV_CUDA_ERROR = 0, 1, 2, 3

c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)
vp = C.c_void_p


class DpvGraph(C.Structure):
    _fields_ = [
        ("n_frames", C.c_int32), ("cells", C.c_int32), ("n_patches", C.c_int64),
        ("n_edges", C.c_int64), ("patch_grid", vp), ("edge_src", vp), ("edge_gpatch", vp),
        ("edge_dst", vp), ("edge_target", vp), ("edge_conf", vp), ("intr", C.c_double * 4),
    ]


class DpvProblemInfo(C.Structure):
    _fields_ = [
        ("n_edges", C.c_int64), ("n_depths", C.c_int64), ("n_free", C.c_int64),
        ("n_keys", C.c_int64), ("n_inc", C.c_int64), ("n_pairs", C.c_int64),
        ("n_segments", C.c_int64), ("n_touched", C.c_int64), ("first_free", C.c_int32),
        ("last_free", C.c_int32), ("scale_degenerate", C.c_int32),
        ("touched_fixed0", C.c_int32), ("device_bytes", C.c_int64),
    ]


class DpvLmParams(C.Structure):
    _fields_ = [("max_iterations", C.c_int32), ("tolerance", C.c_double),
                ("lambda0", C.c_double)]


class DpvPgoReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("initial_objective", C.c_double), ("final_objective", C.c_double),
                ("max_residual_norm", C.c_double), ("final_damping", C.c_double)]


class DpvLmReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32),
        ("initial_objective", C.c_double), ("final_objective", C.c_double),
        ("gradient_norm", C.c_double), ("unconstrained_depths", C.c_int64),
        ("final_damping", C.c_double), ("step_norm", C.c_double),
        ("n_attempts", C.c_int32), ("times_len", C.c_int32),
        ("iteration_times", C.c_double * 64),
    ]


# name -> (restype, argtypes); mirrors include/dpvslam_b200.h one to one
SIGNATURES = {
    "dpv_abi_version": (C.c_int32, []),
    "dpv_last_error": (C.c_char_p, []),
    "dpv_device_info": (C.c_int32, [c_int32_p, c_int32_p, c_int32_p]),
    "dpv_launch_count": (C.c_int64, []),
    "dpv_quat_to_matrix": (C.c_int32, [vp, C.c_int64, vp, vp]),
    "dpv_reproject_grid": (C.c_int32, [vp, vp, vp, vp, vp, vp, C.POINTER(C.c_double), C.c_int64,
                                       C.c_int32, vp, vp, vp, vp, vp]),
    "dpv_problem_create": (C.c_int32, [C.POINTER(DpvGraph), C.c_int32, C.c_int32, vp, C.c_int64,
                                       vp, C.POINTER(vp)]),
    "dpv_problem_destroy": (C.c_int32, [vp]),
    "dpv_problem_get_info": (C.c_int32, [vp, C.POINTER(DpvProblemInfo)]),
    "dpv_problem_array": (C.c_int32, [vp, C.c_char_p, C.POINTER(vp), c_int64_p, c_int32_p]),
    "dpv_gather_depths": (C.c_int32, [vp, vp, vp, vp]),
    "dpv_scatter_depths": (C.c_int32, [vp, vp, vp, vp]),
    "dpv_active_patch_count": (C.c_int32, [vp, C.c_double, c_int64_p, vp]),
    "dpv_residuals": (C.c_int32, [vp, vp, vp, vp, vp, vp, vp]),
    "dpv_objective": (C.c_int32, [vp, vp, vp, vp, vp, vp]),
    "dpv_assemble": (C.c_int32, [vp, vp, vp, vp, vp]),
    "dpv_assemble_edges": (C.c_int32, [vp, vp, vp, vp, vp, vp]),
    "dpv_assemble_rest": (C.c_int32, [vp, vp, vp]),
    "dpv_reduced_system": (C.c_int32, [vp, C.c_double, vp, vp, vp, vp]),
    "dpv_solve": (C.c_int32, [vp, C.c_double, vp, vp, vp, vp]),
    "dpv_solve_backend": (C.c_int32, [vp, C.c_double, C.c_int32, vp, vp, vp, vp]),
    "dpv_back_substitute": (C.c_int32, [vp, C.c_double, vp, vp, vp]),
    "dpv_apply_step": (C.c_int32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "dpv_lm_solve": (C.c_int32, [vp, vp, vp, vp, C.POINTER(DpvLmParams),
                                 C.POINTER(DpvLmReport), vp]),
    "dpv_problem_create_batch": (C.c_int32, [C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp]),
    "dpv_lm_solve_batch": (C.c_int32, [C.c_int32, vp, vp, vp, vp, vp, vp, vp, C.c_int32, vp]),
    "dpv_cholesky_solve": (C.c_int32, [vp, vp, C.c_int64, vp, vp]),
    "dpv_pgo_optimize": (C.c_int32, [C.c_int64, vp, C.c_int64, vp, vp, vp, vp, vp, C.c_int32,
                                     C.c_double, C.c_double, C.POINTER(DpvPgoReport), vp]),
    "dpv_pgo_linearize": (C.c_int32, [C.c_int64, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp]),
    "dpv_fill_flow": (C.c_int32, [C.c_void_p, vp, vp, vp, vp, vp, C.c_int64, vp, vp, vp,
                                  C.c_double, C.c_double, C.c_double, vp, vp, vp]),
    "dpv_reproject_exact": (C.c_int32, [C.c_void_p, vp, vp, vp, vp, C.c_int64, vp, vp]),
    "dpv_visible_landmarks": (C.c_int32, [C.c_int64, C.c_int64, vp, vp, vp, vp, C.c_double,
                                          C.c_double, C.c_double, vp, vp]),
    "dpv_sim3_exp": (C.c_int32, [C.c_int64, vp, vp, vp]),
    "dpv_sim3_log": (C.c_int32, [C.c_int64, vp, vp, vp]),
    "dpv_block_sparse_solve": (C.c_int32, [vp, C.c_int64, C.c_int64, vp, vp, vp, vp, vp]),
    "dpv_problem_spd_info": (C.c_int32, [vp, c_int64_p]),
    "dpv_proximity_detect": (C.c_int32, [vp, C.c_int64, C.c_int64, C.c_double, vp, C.c_int64,
                                         c_int64_p, vp]),
    "dpv_reproject_coords_sel": (C.c_int32, [vp, vp, vp, vp, C.c_double, vp, C.c_int64, vp, vp]),
    "dpv_block_fill_count": (C.c_int32, [vp, C.c_int64, C.c_int64, c_int64_p]),
    "dpv_corr": (C.c_int32, [vp, vp, vp, vp, vp, vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                             C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp]),
    "dpv_corr_ex": (C.c_int32, [vp, C.c_int64, vp, vp, C.c_int64, vp, vp, vp, C.c_int64,
                                C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_int32, C.c_int32, vp, vp]),
    "dpv_corr_ex2": (C.c_int32, [vp, C.c_int64, vp, vp, C.c_int64, vp, vp, vp, C.c_int64,
                                 C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_int32, C.c_int64, vp, vp]),
}

_lib = None


def load(require_gpu: bool = False):
    """Load the shared library (raises NativeUnavailable if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: run `python -m paper_2408_01654_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dpv_abi_version() != 1:
            raise NativeUnavailable("ABI version mismatch")
        _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return _lib


def lib():
    return load(require_gpu=True)


def check(status: int, what: str) -> None:
    if status == DPV_OK:
        return
    msg = _lib.dpv_last_error().decode(errors="replace") if _lib else ""
    if status == DPV_SINGULAR:
        raise SingularSystem(f"{what}: {msg}")
    if status == DPV_BAD_ARGS:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def stream_ptr():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())


class _CudaArray:
    """__cuda_array_interface__ wrapper for a device pointer owned elsewhere."""

    def __init__(self, addr, count, dtype, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (int(count),), "typestr": np.dtype(dtype).str,
            "data": (int(addr), False), "version": 3, "strides": None,
        }


_DTYPES = {0: np.float64, 1: np.int32, 2: np.int64, 3: np.uint8}


def device_view(handle, name: str, owner):
    """Zero-copy torch view of a named array inside a problem handle."""
    import torch
    p = C.c_void_p()
    n = C.c_int64()
    dt = C.c_int32()
    check(lib().dpv_problem_array(handle, name.encode(), C.byref(p), C.byref(n), C.byref(dt)),
          f"problem_array({name})")
    if n.value == 0 or not p.value:
        return torch.zeros(0, dtype=_torch_dtype(dt.value), device="cuda")
    return torch.as_tensor(_CudaArray(p.value, n.value, _DTYPES[dt.value], owner), device="cuda")


def _torch_dtype(code):
    import torch
    return {0: torch.float64, 1: torch.int32, 2: torch.int64, 3: torch.uint8}[code]


SIGNATURES["dpv_avg_pool4"] = (C.c_int32, [vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_int32, vp, vp])
SIGNATURES["dpv_reproject_coords"] = (C.c_int32, [vp, vp, vp, vp, C.c_double, vp, vp])
SIGNATURES["dpv_update_targets"] = (C.c_int32, [vp, vp, vp, vp])
SIGNATURES["dpv_timing_enable"] = (C.c_int32, [C.c_int32])
SIGNATURES["dpv_timing_collect"] = (C.c_int32, [C.c_char_p, C.c_int64, vp, vp, C.c_int32,
                                                c_int32_p])


def timing_enable(on: bool) -> None:
    check(lib().dpv_timing_enable(1 if on else 0), "timing_enable")


def timing_collect() -> dict:
    """{kernel name: (total ms, launches)} since the last collect (synchronises)."""
    cap = 128
    names = C.create_string_buffer(8192)
    ms = (C.c_double * cap)()
    cnt = (C.c_int64 * cap)()
    n = C.c_int32()
    check(lib().dpv_timing_collect(names, 8192, C.cast(ms, vp), C.cast(cnt, vp), cap, C.byref(n)),
          "timing_collect")
    keys = names.value.decode().split("\n")[:n.value]
    return {k: (ms[i], int(cnt[i])) for i, k in enumerate(keys)}
SIGNATURES["dpv_problem_create_ex"] = (C.c_int32, [C.POINTER(DpvGraph), C.c_int32, C.c_int32, vp,
                                                   C.c_int64, vp, C.c_int64, vp, C.POINTER(vp)])
SIGNATURES["dpv_problem_set_gauge"] = (C.c_int32, [vp, C.c_int32, C.c_int32])
SIGNATURES["dpv_problem_plan_info"] = (C.c_int32, [vp, c_int32_p, c_int64_p, c_int64_p,
                                                   C.POINTER(C.c_double)])


def plan_info(handle) -> dict:
    d = C.c_int32()
    t = C.c_int64()
    u = C.c_int64()
    f = C.c_double()
    check(lib().dpv_problem_plan_info(handle, C.byref(d), C.byref(t), C.byref(u), C.byref(f)),
          "plan_info")
    return {"dense": bool(d.value), "tiles": int(t.value), "update_tiles": int(u.value),
            "update_flops": float(f.value)}


def spd_info(handle) -> dict:
    """Sparse band+border factor plan (dpv_problem_spd_info)."""
    v = (C.c_int64 * 9)()
    check(lib().dpv_problem_spd_info(handle, C.cast(v, c_int64_p)), "spd_info")
    names = ("n", "chains", "band_tiles", "tile_bandwidth", "border_poses", "border_rows",
             "level2_tiles", "factor_ctas", "model_us")
    return {k: int(v[i]) for i, k in enumerate(names)}
