"""ctypes binding of the C-ABI declared in include/ddsg_b200.h.

There is no fallback: if libddsg_b200.so is missing the import fails loudly
(build it with ``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# DDSG_B200_LIB selects another in-tree build of the same library (A/B
# measurements of build-time variants, e.g. libddsg_b200_c16.so)
LIB_PATH = _PKG / os.environ.get("DDSG_B200_LIB", "libddsg_b200.so")
WL_PATH = _PKG / "libddsg_workloads.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: the DDSG CUDA library has not been built "
        "(run __graft_entry__.build()); there is no CPU fallback"
    )

lib = C.CDLL(str(LIB_PATH))

# status codes
OK, INVALID_ARGUMENT, DOMAIN_ERROR, CUDA_ERROR, NCCL_ERROR, OUT_OF_MEMORY, BUILD_ERROR, OUT_OF_RANGE = range(8)
ZERO_BOUNDARY, MODIFIED_LINEAR = 0, 1
NORM_INF, NORM_L2 = 0, 1
EVAL_EXACT, EVAL_FAST = 0, 1

BATCH_EVALUATOR = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double), C.c_void_p)
NODE_EVALUATOR = C.CFUNCTYPE(C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double), C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class RefineStatsC(C.Structure):
    """ddsg_refine_stats (include/ddsg_b200.h)."""

    _fields_ = [("new_nodes", C.c_int64), ("rounds", C.c_int64), ("gathered_bytes", C.c_int64),
                ("target_s", C.c_double), ("hierarchize_s", C.c_double), ("allgather_s", C.c_double)]

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double
_pd = C.c_void_p  # raw pointers (host numpy or device)

# name: (restype, argtypes) — mirrors include/ddsg_b200.h one to one
SIGNATURES = {
    "ddsg_last_error": (C.c_char_p, []),
    "ddsg_device_count": (_i, []),
    "ddsg_grid_create": (_i, [_i, _i, _i, _i, _d, _i64, _p, _p, C.POINTER(_p)]),
    "ddsg_grid_build": (_i, [_i, _i, _i, _i, _d, _i, _p, _p, C.POINTER(_p)]),
    "ddsg_last_build_point": (_i, [_p, _i]),
    "ddsg_grid_append": (_i, [_p, _i64, _p, _p]),
    "ddsg_hierarchize": (_i, [_p, _i64, _p, _p, _p]),
    "ddsg_grid_destroy": (_i, [_p]),
    "ddsg_hierarchize_host": (_i, [_p, _i64, _p, _p, _p]),
    "ddsg_grid_refine_candidates": (_i, [_p, _i, C.POINTER(_i64), _p]),
    "ddsg_grid_info": (_i, [_p, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_d), C.POINTER(_i64)]),
    "ddsg_grid_nodes": (_i, [_p, _p, _p]),
    "ddsg_grid_quadrature": (_i, [_p, _p]),
    "ddsg_grid_find": (_i, [_p, _p, C.POINTER(_i64)]),
    "ddsg_eval_grid": (_i, [_p, _pd, _i64, _pd, C.POINTER(_i64), _p]),
    "ddsg_hdmr_create": (_i, [_i, _i, _p, _i, _p, _p, _p, _p, C.POINTER(_p)]),
    "ddsg_hdmr_destroy": (_i, [_p]),
    "ddsg_hdmr_info": (_i, [_p, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i64)]),
    "ddsg_eval_hdmr": (_i, [_p, _pd, _i64, _pd, C.POINTER(_i64), _p]),
    "ddsg_hdmr_quadrature": (_i, [_p, _p]),
    "ddsg_grid_set_eval_mode": (_i, [_p, _i]),
    "ddsg_hdmr_set_eval_mode": (_i, [_p, _i]),
    "ddsg_last_eval_stats": (_i, [C.POINTER(_i64), C.POINTER(_d), C.POINTER(_d)]),
    "ddsg_hdmr_kernel_path": (_i, [_p, C.POINTER(_i)]),
    "ddsg_measure_fp64_peak": (_i, [C.POINTER(_d), C.POINTER(_d)]),
    "ddsg_hdmr_support": (_i, [_p, _pd, _i64, _pd, _pd, _p]),
    "ddsg_grid_support": (_i, [_p, _pd, _i64, _pd, _pd, _p]),
    "ddsg_uniform_points": (None, [C.c_uint64, _i64, _i, _p]),
    "ddsg_uniform_point_blocks": (None, [C.c_uint64, _i64, _i64, _i64, _i, _p]),
    "ddsg_hdmr_slot": (_i, [_p, _i, C.POINTER(_i), _p, C.POINTER(C.c_int32), C.POINTER(_p)]),
    "ddsg_grid_from_json": (_i, [C.c_char_p, _i64, C.POINTER(_p)]),
    "ddsg_grid_to_json": (_i, [_p, _p, _i64, C.POINTER(_i64)]),
    "ddsg_hdmr_from_json": (_i, [C.c_char_p, _i64, C.POINTER(_p)]),
    "ddsg_hdmr_to_json": (_i, [_p, _p, _i64, C.POINTER(_i64)]),
    "ddsg_hdmr_set_document": (_i, [_p, _i, _p, _i, _p, _p, _p]),
    "ddsg_hdmr_document": (_i, [_p, C.POINTER(_i), _p, _p, C.POINTER(_i), C.POINTER(_i64), _p, _p, C.POINTER(_i), _p]),
    "ddsg_refine_step": (_i, [_p, _i, _p, _p, _p, _i, _i, _p, _p, _i, _p]),
    "ddsg_refine_step_nccl": (_i, [_p, _i, _p, _p, _p, _p, _i, _i, _p, _p]),
    "ddsg_workspace_create": (_i, [C.POINTER(_p)]),
    "ddsg_workspace_destroy": (_i, [_p]),
    "ddsg_eval_hdmr_ws": (_i, [_p, _p, _pd, _i64, _pd, C.POINTER(_i64), C.POINTER(C.c_uint64)]),
    "ddsg_eval_grid_ws": (_i, [_p, _p, _pd, _i64, _pd, C.POINTER(_i64)]),
    "ddsg_eval_hdmr_rows": (_i, [_p, _p, _p, _i64, _p, C.POINTER(_i64)]),
    "ddsg_irbc_refresh_derived": (_i, [_p, _i]),
    "ddsg_irbc_steady_state_lambda": (_i, [_p, C.POINTER(_d)]),
    "ddsg_irbc_foc_residuals": (_i, [_p, _p, _p, _i64, _pd, _pd, _pd, _pd, _pd, C.POINTER(_i64), _p]),
    "ddsg_irbc_foc_jacobian": (_i, [_p, _p, _p, _i64, _pd, _pd, _pd, _pd, _d, _pd, C.POINTER(_i64), _p]),
    "ddsg_irbc_euler_errors": (_i, [_p, _p, _p, _i64, _pd, _pd, C.POINTER(_d), C.POINTER(_d), C.POINTER(C.c_uint64),
                                    C.POINTER(_i64), _p]),
}


class IrbcParamsC(C.Structure):
    """ddsg_irbc_params (include/ddsg_b200.h)."""

    _fields_ = [("countries", _i), ("variant", _i), ("beta", _d), ("alpha", _d), ("delta", _d), ("sigma", _d),
                ("rho_a", _d), ("phi_adj", _d), ("gamma_base", _d), ("lna_half_width", _d), ("k_lo", _d),
                ("k_hi", _d), ("A", _d), ("gamma", C.POINTER(_d)), ("tau", C.POINTER(_d))]

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return lib.ddsg_last_error().decode()


_wl = None


def workloads():
    """The synthetic-workload library (target functions of the configs)."""
    global _wl
    if _wl is None:
        if not WL_PATH.exists():
            raise ImportError(f"{WL_PATH} is missing (run __graft_entry__.build())")
        _wl = C.CDLL(str(WL_PATH))
        _wl.wl_cut_new.restype = C.c_void_p
        _wl.wl_cut_new.argtypes = [C.c_void_p, C.c_void_p, _i, _i, _i, _p, _p]
        _wl.wl_cut_free.argtypes = [C.c_void_p]
        _wl.wl_config_pairs.restype = _i
        _wl.wl_config_pairs.argtypes = [_i, _p]
    return _wl


def wl_fn(name: str) -> int:
    """Address of a C target function in the workloads library."""
    return C.cast(getattr(workloads(), name), C.c_void_p).value
