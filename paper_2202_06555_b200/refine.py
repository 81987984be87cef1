"""One adaptive refinement step of a set of component grids, distributed over
ranks (the path's only collective).

For every grid, the new batch is the reference's next build batch
(`SparseGridFunction.refine_candidates`, sparse_grid.hpp:215-254).  Batches
are hierarchized group by group in ascending level sum (bases
of equal level sum vanish at each other's nodes, so a group's nodes are
independent, but a group needs every lower group appended first).  Per round,
the new nodes of all grids are split evenly (padded) across the ranks; each
rank evaluates the target and hierarchizes its share on its own GPU
(`ddsg_hierarchize`, exact), the surplus rows are all-gathered (NCCL over
NVLink on GPU ranks, gloo in the CPU tests) and every rank appends the whole
group in batch order — grids stay replicated and bit-identical on every rank,
and equal to the reference's `build` at the next level.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from .ddsg import SparseGridFunction


@dataclass
class RefineStats:
    new_nodes: int = 0
    rounds: int = 0
    gathered_bytes: int = 0
    hierarchize_s: float = 0.0  # GPU (or host) hierarchization of this rank's share
    target_s: float = 0.0       # the caller's target evaluations (host model code)
    allgather_s: float = 0.0
    per_round: List[int] = field(default_factory=list)


def coords_of(keys: np.ndarray) -> np.ndarray:
    """Grid coordinates i * 2^-l of heap keys (grid_index.hpp:41-44), exact."""
    keys = np.asarray(keys, dtype=np.uint32)
    lm1 = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64)  # l - 1
    index = 2 * (keys.astype(np.int64) - (np.int64(1) << lm1)) + 1
    return index.astype(np.float64) * np.ldexp(1.0, -(lm1 + 1))


def _level_sums(keys: np.ndarray) -> np.ndarray:
    lv = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64) + 1
    return lv.sum(axis=1)


def _all_gather_rows(local: np.ndarray, rows_per_rank: int, m: int, dist, device: str):
    """All-gather [rows_per_rank][m] float64 blocks; returns [world*rows_per_rank][m]."""
    import torch

    world = dist.get_world_size()
    t = torch.from_numpy(np.ascontiguousarray(local)).to(device)
    if device.startswith("cuda"):
        out = torch.empty((world * rows_per_rank, m), dtype=torch.float64, device=device)
        dist.all_gather_into_tensor(out, t)  # ncclAllGather over NVLink
        return out.cpu().numpy()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return torch.cat(parts).numpy()


def refine_step(grids: Sequence[SparseGridFunction], level_sums: Sequence[int],
                f_eval: Callable[[int, np.ndarray], np.ndarray], dist=None, device: bool = True,
                comm_device: Optional[str] = None) -> RefineStats:
    """Refines every grid by one level-sum step.

    grids:      component grids (same out_dim), replicated on every rank
    level_sums: per grid, the level sum s whose significant nodes get children
    f_eval:     f_eval(grid_index, xs[count][dim]) -> values[count][m]; called
                only for this rank's share of the new nodes
    dist:       torch.distributed (initialised) or None for a single process
    device:     hierarchize on the GPU (True) or on the host (False)
    """
    stats = RefineStats()
    m = grids[0].out_dim
    rank = dist.get_rank() if dist is not None else 0
    world = dist.get_world_size() if dist is not None else 1
    if comm_device is None:
        comm_device = "cuda" if device else "cpu"
    batches = [g.refine_candidates(s) for g, s in zip(grids, level_sums)]
    groups = []
    for keys in batches:
        if len(keys) == 0:
            groups.append([])
            continue
        ls = _level_sums(keys)
        # the batch is sorted by (level sum, key): groups are contiguous
        groups.append([keys[ls == v] for v in np.unique(ls)])
    n_rounds = max((len(g) for g in groups), default=0)
    for r in range(n_rounds):
        items = []  # (grid index, keys) of this round, in grid order
        for gi, gr in enumerate(groups):
            if r < len(gr):
                items.append((gi, gr[r]))
        total = sum(len(k) for _, k in items)
        if total == 0:
            continue
        q = (total + world - 1) // world
        lo, hi = rank * q, min(total, (rank + 1) * q)
        local = np.zeros((q, m), dtype=np.float64)
        off = 0
        for gi, keys in items:
            a, b = max(lo, off), min(hi, off + len(keys))
            if a < b:
                sub = keys[a - off:b - off]
                xs = coords_of(sub)
                t0 = time.perf_counter()
                fv = np.asarray(f_eval(gi, xs), dtype=np.float64).reshape(len(sub), m)
                stats.target_s += time.perf_counter() - t0
                if not np.all(np.isfinite(fv)):
                    raise FloatingPointError(f"refine_step: non-finite target value on grid {gi}")
                t0 = time.perf_counter()
                local[a - lo:b - lo] = grids[gi].hierarchize(sub, fv, device=device)
                stats.hierarchize_s += time.perf_counter() - t0
            off += len(keys)
        t0 = time.perf_counter()
        if dist is not None:
            allrows = _all_gather_rows(local, q, m, dist, comm_device)[:total]
            stats.gathered_bytes += world * q * m * 8
        else:
            allrows = local[:total]
        stats.allgather_s += time.perf_counter() - t0
        off = 0
        for gi, keys in items:
            grids[gi].append(keys, allrows[off:off + len(keys)])
            off += len(keys)
        stats.new_nodes += total
        stats.rounds += 1
        stats.per_round.append(total)
    return stats
