"""TEST INFRASTRUCTURE (bench.py's reference arm and CPU-baseline leg): the
BASELINE HDMR configs built and evaluated by the REFERENCE alone.

Everything here goes through oracle/_ref/libddsg_ref*.so -- the unmodified
reference headers compiled in place (oracle/Makefile), which also link the
synthetic targets (csrc_workloads/workloads.c, compiled like
libddsg_workloads.so).  No product library is loaded: the config data come
from paper_2202_06555_b200/configs.py loaded by path (the package __init__
would load libddsg_b200.so).

  family     all first-order indices + the config's pairs (wl_config_pairs)
  b          oracle::b_coefficients_bruteforce (proj/tests/oracles.hpp:72-81)
  f_anchor   the target at the centre anchor (hdmr.hpp:380-382)
  cut grids  SparseGridFunction::build (sparse_grid.hpp:84-108) of the cut
             evaluator (hdmr.hpp cut_evaluator semantics, wl_cut_eval)
  points     oracle::uniform_points (oracles.hpp:45-53) per block of the
             blocked stream (block b: mt19937_64(seed + b))
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as O  # noqa: E402

BLOCK_POINTS = 1 << 14  # point block of the bench's seeded stream (bench.py, ddsg_uniform_point_blocks)


def configs():
    spec = importlib.util.spec_from_file_location("_ddsg_configs", ROOT / "paper_2202_06555_b200" / "configs.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_ddsg_configs"] = mod  # dataclasses resolve annotations through sys.modules
    spec.loader.exec_module(mod)
    return mod.CONFIGS


def use_library(path: Path):
    """Selects which oracle/_ref build oracle_lib binds (generic or x86-64-v3)."""
    O._ref = None
    O.REF_PATH = Path(path)
    lib = O.ref()
    if lib is None:
        raise RuntimeError(f"{path} missing")
    lib.wl_cut_new.restype = C.c_void_p
    lib.wl_cut_new.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.wl_cut_free.argtypes = [C.c_void_p]
    lib.wl_config_pairs.restype = C.c_int
    lib.wl_config_pairs.argtypes = [C.c_int, C.c_void_p]
    lib.ref_b_coefficients.restype = C.c_int
    lib.ref_b_coefficients.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


def _fn(lib, name: str) -> int:
    return C.cast(getattr(lib, name), C.c_void_p).value


def family(lib, cfg):
    cfg_id = 4 if cfg.d == 100 else 5
    pairs = np.zeros(2 * 400, dtype=np.int32)
    n_pairs = lib.wl_config_pairs(cfg_id, pairs.ctypes.data)
    fam = [()] + [(k,) for k in range(cfg.d)]
    fam += sorted({(int(pairs[2 * r]), int(pairs[2 * r + 1])) for r in range(n_pairs)})
    return fam


def b_coefficients(lib, fam):
    order = np.array([len(u) for u in fam], dtype=np.int32)
    dims = np.array([v for u in fam for v in u] or [0], dtype=np.int32)
    b = np.zeros(len(fam), dtype=np.int32)
    assert lib.ref_b_coefficients(len(fam), order.ctypes.data, dims.ctypes.data, b.ctypes.data) == 0
    return [int(v) for v in b]


def build_hdmr(cfg, lib):
    """(RefHdmr, f_anchor, family, b): the config's VectorizedDdsg, every cut
    grid built by the reference's SparseGridFunction::build."""
    fam = family(lib, cfg)
    b = b_coefficients(lib, fam)
    anchor = np.full(cfg.d, 0.5)
    fa = np.empty(cfg.m)
    f = getattr(lib, cfg.target)
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    f(anchor.ctypes.data, 1, fa.ctypes.data, None)
    f_addr, cut_addr = _fn(lib, cfg.target), _fn(lib, "wl_cut_eval")
    grids = []
    for u in fam:
        if not u:
            grids.append(None)
            continue
        dims = np.array(u, dtype=np.int32)
        cut = lib.wl_cut_new(f_addr, None, cfg.d, cfg.m, len(u), dims.ctypes.data, anchor.ctypes.data)
        lvl = cfg.level_1d if len(u) == 1 else cfg.level_2d
        eps = cfg.eps_1d if len(u) == 1 else cfg.eps_2d
        rc, g = O.ref_build(len(u), cfg.m, cfg.mode, lvl, eps, cut_addr, C.c_void_p(cut))
        lib.wl_cut_free(C.c_void_p(cut))
        if rc != 0:
            raise RuntimeError(f"reference build of cut {u} failed: {g}")
        grids.append(g)
    return O.RefHdmr(cfg.d, cfg.m, fa, list(zip(fam, b)), grids), fa, fam, b


def points(lib, cfg, first: int, n: int, block_points: int = BLOCK_POINTS):
    """Points [first, first + n) of the bench's blocked seeded stream."""
    out = np.empty((n, cfg.d))
    b0, b1 = first // block_points, (first + n - 1) // block_points
    for blk in range(b0, b1 + 1):
        lo, hi = max(first, blk * block_points), min(first + n, (blk + 1) * block_points)
        buf = np.empty((hi - blk * block_points, cfg.d))
        lib.ref_uniform_points(cfg.d, buf.shape[0], (cfg.seed + blk) & ((1 << 64) - 1), buf.ctypes.data)
        out[lo - first: hi - first] = buf[lo - blk * block_points:]
    return out
