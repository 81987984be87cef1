"""Synthetic workloads of BASELINE.json's five configs.

Every grid is built by this package's own builder (ddsg_grid_build, the
reference's build algorithm) from C target functions in
libddsg_workloads.so; HDMR configs are assembled from cut grids through
VectorizedDdsg.compile (DdsgFunction::from_parts + compile, hdmr.hpp:307-325,
ddsg_eval.hpp:40-74) with a center anchor.  Choices BASELINE.json leaves open
are fixed here and recorded in DESIGN.md §Workloads.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .configs import CONFIGS, Config  # noqa: F401  (re-exported)
from .ddsg import MODIFIED_LINEAR, ZERO_BOUNDARY, SparseGridFunction, VectorizedDdsg


def telescoping_b(family: List[Tuple[int, ...]]) -> List[int]:
    """b_i = sum over family members u >= i of (-1)^(|u|-|i|)
    (hdmr.hpp:339-355 finalize_coefficients; family includes the empty index)."""
    sets = [frozenset(u) for u in family]
    out = []
    for i, si in enumerate(sets):
        b = 0
        for u, su in enumerate(sets):
            if si <= su:
                b += 1 if (len(su) - len(si)) % 2 == 0 else -1
        out.append(b)
    return out


def build_grid(cfg: Config) -> SparseGridFunction:
    return SparseGridFunction.build(N.wl_fn(cfg.target), cfg.d, cfg.m, cfg.max_level, cfg.eps_gamma, cfg.mode)


def hdmr_family(cfg: Config) -> List[Tuple[int, ...]]:
    wl = N.workloads()
    if cfg.kind != "hdmr":
        raise ValueError("not an HDMR config")
    cfg_id = 4 if cfg.d == 100 else 5
    pairs = np.zeros(2 * 400, dtype=np.int32)
    n_pairs = wl.wl_config_pairs(cfg_id, pairs.ctypes.data)
    fam: List[Tuple[int, ...]] = [()]
    fam += [(k,) for k in range(cfg.d)]
    fam += sorted({(int(pairs[2 * r]), int(pairs[2 * r + 1])) for r in range(n_pairs)})
    return fam


@dataclass
class HdmrParts:
    d: int
    m: int
    f_anchor: np.ndarray
    slots: list = field(default_factory=list)  # (dims, b, SparseGridFunction or None)


def build_hdmr_parts(cfg: Config, build_grids: bool = True) -> HdmrParts:
    """The config's family, b, anchor values and (build_grids) cut grids;
    build_grids=False leaves every grid None (the receivers of a broadcast,
    see broadcast_hdmr_parts)."""
    wl = N.workloads()
    fam = hdmr_family(cfg)
    b = telescoping_b(fam)
    anchor = np.full(cfg.d, 0.5)
    fa = np.empty(cfg.m)
    fn = getattr(wl, cfg.target)
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    fn(anchor.ctypes.data, 1, fa.ctypes.data, None)
    parts = HdmrParts(cfg.d, cfg.m, fa)
    f_addr = N.wl_fn(cfg.target)
    cut_addr = N.wl_fn("wl_cut_eval")

    def build_cut(u):
        dims = np.array(u, dtype=np.int32)
        cut = wl.wl_cut_new(f_addr, None, cfg.d, cfg.m, len(u), dims.ctypes.data, anchor.ctypes.data)
        try:
            lvl = cfg.level_1d if len(u) == 1 else cfg.level_2d
            eps = cfg.eps_1d if len(u) == 1 else cfg.eps_2d
            return SparseGridFunction.build(cut_addr, len(u), cfg.m, lvl, eps, cfg.mode, ctx=cut)
        finally:
            wl.wl_cut_free(C.c_void_p(cut))

    # the cut builds are independent host C calls (ctypes releases the GIL;
    # the target's tables were initialised by the anchor evaluation above)
    import concurrent.futures as cf

    if not build_grids:
        parts.slots.extend((u, bu, None) for u, bu in zip(fam, b))
        return parts
    with cf.ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        grids = list(ex.map(lambda u: build_cut(u) if u else None, fam))
    parts.slots.extend((u, bu, g) for u, bu, g in zip(fam, b, grids))
    return parts


def broadcast_hdmr_parts(cfg: Config, dist, device: str, level_1d: Optional[int] = None) -> HdmrParts:
    """Build once, broadcast: rank 0 builds every cut grid; the node keys and
    surplus rows go to the other ranks in three broadcasts (counts, keys,
    surpluses; NCCL over NVLink for CUDA tensors) and every rank assembles the
    same grids with from_nodes (identical stored order and bits).
    level_1d overrides the 1-d cut level (the bench builds one level short
    and refines)."""
    import dataclasses

    import torch

    rank = dist.get_rank()
    c = dataclasses.replace(cfg, level_1d=level_1d) if level_1d is not None else cfg
    parts = build_hdmr_parts(c, build_grids=(rank == 0))
    idx = [i for i, (u, _, _) in enumerate(parts.slots) if u]
    counts = torch.zeros(len(idx), dtype=torch.int64, device=device)
    if rank == 0:
        counts.copy_(torch.tensor([parts.slots[i][2].size() for i in idx], dtype=torch.int64))
    dist.broadcast(counts, 0)
    cnt = counts.cpu().numpy()
    k_tot = int(sum(int(n) * len(parts.slots[i][0]) for n, i in zip(cnt, idx)))
    s_tot = int(cnt.sum()) * c.m
    keys = torch.empty(k_tot, dtype=torch.int32, device=device)
    sur = torch.empty(s_tot, dtype=torch.float64, device=device)
    if rank == 0:
        ks, ss = [], []
        for i in idx:
            k, s = parts.slots[i][2].nodes()
            ks.append(k.reshape(-1).view(np.int32))
            ss.append(s.reshape(-1))
        keys.copy_(torch.from_numpy(np.concatenate(ks)))
        sur.copy_(torch.from_numpy(np.concatenate(ss)))
    dist.broadcast(keys, 0)
    dist.broadcast(sur, 0)
    if rank != 0:
        kh = keys.cpu().numpy().view(np.uint32)
        sh = sur.cpu().numpy()
        ko = so = 0
        slots = list(parts.slots)
        for n, i in zip(cnt, idx):
            u, bu, _ = slots[i]
            k = len(u)
            lvl, eps = (c.level_1d, c.eps_1d) if k == 1 else (c.level_2d, c.eps_2d)
            g = SparseGridFunction.from_nodes(k, c.m, lvl, eps, c.mode, kh[ko:ko + n * k].reshape(n, k),
                                              sh[so:so + n * c.m].reshape(n, c.m))
            ko += int(n) * k
            so += int(n) * c.m
            slots[i] = (u, bu, g)
        parts.slots = slots
    return parts


class GridTarget:
    """A plain-grid config's target (configs 1-3) as a numpy batch function
    xs[n][d] -> values[n][m] (the C evaluator the builds use)."""

    def __init__(self, cfg: Config):
        self.cfg = cfg
        self._fn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)(N.wl_fn(cfg.target))

    def __call__(self, xs: np.ndarray) -> np.ndarray:
        xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1, self.cfg.d)
        out = np.empty((xs.shape[0], self.cfg.m))
        if xs.shape[0] and self._fn(xs.ctypes.data, xs.shape[0], out.ctypes.data, None) != 0:
            raise RuntimeError(f"{self.cfg.target} failed")
        return out


class CutTarget:
    """The config target restricted to the cut through the center anchor along
    `dims` (hdmr.hpp:248-259), as a C evaluator (address + ctx) and a numpy
    batch function."""

    def __init__(self, cfg: Config, dims: Tuple[int, ...]):
        wl = N.workloads()
        self.cfg, self.dims = cfg, tuple(dims)
        self._dims = np.array(dims, dtype=np.int32)
        self._anchor = np.full(cfg.d, 0.5)
        self.ctx = wl.wl_cut_new(N.wl_fn(cfg.target), None, cfg.d, cfg.m, len(dims), self._dims.ctypes.data,
                                 self._anchor.ctypes.data)
        if not self.ctx:
            raise ValueError(f"cut of {len(dims)} dims not supported (1..16)")
        self.addr = N.wl_fn("wl_cut_eval")
        self._fn = wl.wl_cut_eval
        self._fn.restype = C.c_int
        self._fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]

    def __call__(self, xs: np.ndarray) -> np.ndarray:
        xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1, len(self.dims))
        out = np.empty((xs.shape[0], self.cfg.m))
        if xs.shape[0]:
            self._fn(xs.ctypes.data, xs.shape[0], out.ctypes.data, C.c_void_p(self.ctx))
        return out

    def __del__(self):
        if getattr(self, "ctx", None):
            N.workloads().wl_cut_free(C.c_void_p(self.ctx))
            self.ctx = None


def build_cut_grid(cfg: Config, dims: Tuple[int, ...], level: int, eps: float) -> SparseGridFunction:
    cut = CutTarget(cfg, dims)
    return SparseGridFunction.build(cut.addr, len(dims), cfg.m, level, eps, cfg.mode, ctx=cut.ctx)


def build_hdmr(cfg: Config) -> Tuple[VectorizedDdsg, HdmrParts]:
    parts = build_hdmr_parts(cfg)
    return VectorizedDdsg.compile(parts.d, parts.m, parts.f_anchor, parts.slots), parts


def points(cfg: Config, n: Optional[int] = None, seed: Optional[int] = None) -> np.ndarray:
    from .ddsg import uniform_points

    return uniform_points(cfg.seed if seed is None else seed, cfg.n_points if n is None else n, cfg.d)


# ------------------------------------------------------ IRBC policy targets

class IrbcPolicyTarget:
    """wl_irbc_policy (workloads.c): a policy-shaped target on the canonical
    state cube of an N-country IRBC model, for the batched callers
    (SURVEY.md §8(f) rows 2-3).  ``steady=True`` is the reference tests'
    steady policy (k' = k, mu = 0, lambda = lam0; test_irbc.cpp:14-24)."""

    def __init__(self, countries: int, nonsmooth: bool = False, steady: bool = False, n_pairs: int = 0,
                 seed: int = 20220213, delta: float = 0.01, k_lo: float = 0.5, k_hi: float = 1.5,
                 lna_half_width: float = 0.4, lam0: float = 1.0):
        wl = N.workloads()
        wl.wl_irbc_new.restype = C.c_void_p
        wl.wl_irbc_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_double]
        wl.wl_irbc_free.argtypes = [C.c_void_p]
        wl.wl_irbc_pairs.restype = C.c_int
        wl.wl_irbc_pairs.argtypes = [C.c_void_p, C.c_void_p]
        self.countries = countries
        self.d = 2 * countries
        self.m = 2 * countries + 1 if nonsmooth else countries + 1
        self.ctx = wl.wl_irbc_new(countries, int(nonsmooth), int(steady), n_pairs, seed, delta, k_lo, k_hi,
                                  lna_half_width, lam0)
        if not self.ctx:
            raise ValueError("wl_irbc_new: bad arguments")
        pairs = np.zeros(2 * max(n_pairs, 1), dtype=np.int32)
        n = wl.wl_irbc_pairs(self.ctx, pairs.ctypes.data)
        self.pairs = [(int(pairs[2 * r]), int(pairs[2 * r + 1])) for r in range(n)]
        self.addr = N.wl_fn("wl_irbc_policy")
        self._fn = wl.wl_irbc_policy
        self._fn.restype = C.c_int
        self._fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]

    def __call__(self, xs: np.ndarray) -> np.ndarray:
        xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1, self.d)
        out = np.empty((xs.shape[0], self.m))
        if xs.shape[0]:
            self._fn(xs.ctypes.data, xs.shape[0], out.ctypes.data, C.c_void_p(self.ctx))
        return out

    def __del__(self):
        if getattr(self, "ctx", None):
            N.workloads().wl_irbc_free(C.c_void_p(self.ctx))
            self.ctx = None


def build_policy_grid(target: IrbcPolicyTarget, max_level: int, eps: float = 0.0,
                      mode: int = MODIFIED_LINEAR) -> SparseGridFunction:
    """The policy as one plain sparse grid on [0,1]^(2N)."""
    return SparseGridFunction.build(target.addr, target.d, target.m, max_level, eps, mode, ctx=target.ctx)


def build_policy_hdmr(target: IrbcPolicyTarget, level_1d: int, level_2d: int, eps_1d: float = 0.0,
                      eps_2d: float = 0.0, mode: int = MODIFIED_LINEAR) -> Tuple[VectorizedDdsg, HdmrParts]:
    """The policy as a cut-HDMR (center anchor): all 1-d cuts plus the
    target's pair cuts, like configs 4-5."""
    wl = N.workloads()
    fam: List[Tuple[int, ...]] = [()] + [(k,) for k in range(target.d)] + sorted(set(target.pairs))
    b = telescoping_b(fam)
    anchor = np.full(target.d, 0.5)
    fa = target(anchor)[0]
    parts = HdmrParts(target.d, target.m, fa)
    cut_addr = N.wl_fn("wl_cut_eval")
    for u, bu in zip(fam, b):
        if not u:
            parts.slots.append((u, bu, None))
            continue
        dims = np.array(u, dtype=np.int32)
        cut = wl.wl_cut_new(target.addr, target.ctx, target.d, target.m, len(u), dims.ctypes.data,
                            anchor.ctypes.data)
        try:
            lvl, eps = (level_1d, eps_1d) if len(u) == 1 else (level_2d, eps_2d)
            g = SparseGridFunction.build(cut_addr, len(u), target.m, lvl, eps, mode, ctx=cut)
        finally:
            wl.wl_cut_free(C.c_void_p(cut))
        parts.slots.append((u, bu, g))
    return VectorizedDdsg.compile(parts.d, parts.m, parts.f_anchor, parts.slots), parts
