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
and equal to the reference's `build` at the next level.  The orchestration
is native (C-ABI ddsg_refine_step, csrc/refine.cu); this module only adapts
the caller's target and torch.distributed to it.
"""
from __future__ import annotations

from dataclasses import dataclass
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
    collective: str = "none"


def coords_of(keys: np.ndarray) -> np.ndarray:
    """Grid coordinates i * 2^-l of heap keys (grid_index.hpp:41-44), exact."""
    keys = np.asarray(keys, dtype=np.uint32)
    lm1 = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64)  # l - 1
    index = 2 * (keys.astype(np.int64) - (np.int64(1) << lm1)) + 1
    return index.astype(np.float64) * np.ldexp(1.0, -(lm1 + 1))


class _DeviceArray:
    """A raw device allocation as a __cuda_array_interface__ object (so torch
    can wrap the library's device buffers without copying)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def _nccl_comm(dist):
    """torch's ncclComm_t of the default group, or None (gloo, no NCCL)."""
    try:
        import torch

        if dist.get_backend() != "nccl":
            return None
        pg = dist.distributed_c10d._get_default_group()
        backend = pg._get_backend(torch.device("cuda"))
        ptr = int(backend._comm_ptr())
        if ptr == 0:  # NCCL communicators are created lazily by the first collective
            dist.all_reduce(torch.zeros(1, device="cuda"))
            torch.cuda.synchronize()
            ptr = int(backend._comm_ptr())
        return ptr or None
    except Exception:
        return None


def refine_step(grids: Sequence[SparseGridFunction], level_sums: Sequence[int],
                f_eval: Callable[[int, np.ndarray], np.ndarray], dist=None, device: bool = True,
                comm_device: Optional[str] = None) -> RefineStats:
    """Refines every grid by one level-sum step (C-ABI ddsg_refine_step /
    ddsg_refine_step_nccl: the orchestration is native).

    grids:      component grids (same out_dim), replicated on every rank
    level_sums: per grid, the level sum s whose significant nodes get children
    f_eval:     f_eval(grid_index, xs[count][dim]) -> values[count][m]; called
                only for this rank's share of the new nodes
    dist:       torch.distributed (initialised) or None for a single process.
                With the NCCL backend the library all-gathers the device rows
                itself over torch's communicator (ncclAllGather, no host
                bounce); otherwise through a torch.distributed all-gather
                (device tensors wrapping the library's buffers, or host
                arrays for gloo with device=False).
    device:     hierarchize on the GPU (True) or on the host (False)
    """
    import ctypes as C

    from . import _native as N
    from .ddsg import _check

    m = grids[0].out_dim
    dims = [g.dim for g in grids]
    rank = dist.get_rank() if dist is not None else 0
    world = dist.get_world_size() if dist is not None else 1
    errors: List[BaseException] = []

    def node_eval(gi, xs, count, out, ctx):
        try:
            x = np.ctypeslib.as_array(xs, shape=(count, dims[gi])).copy()
            y = np.asarray(f_eval(gi, x), dtype=np.float64).reshape(count, m)
            np.ctypeslib.as_array(out, shape=(count, m))[:] = y
            return 0
        except BaseException as e:  # surfaced after the C call
            errors.append(e)
            return 1

    def allgather(send, recv, nbytes, ctx):
        try:
            import torch

            n = nbytes // 8
            if device:
                ts = torch.as_tensor(_DeviceArray(send, n), device="cuda")
                tr = torch.as_tensor(_DeviceArray(recv, n * world), device="cuda")
                if dist.get_backend() == "nccl":
                    dist.all_gather_into_tensor(tr, ts)
                else:  # gloo: host staging of the device rows
                    parts = [torch.empty(n, dtype=torch.float64) for _ in range(world)]
                    dist.all_gather(parts, ts.cpu())
                    tr.copy_(torch.cat(parts))
                torch.cuda.synchronize()
            else:
                ts = torch.from_numpy(np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_double)), shape=(n,)).copy())
                parts = [torch.empty_like(ts) for _ in range(world)]
                dist.all_gather(parts, ts)
                np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_double)), shape=(n * world,))[:] = \
                    torch.cat(parts).numpy()
            return 0
        except BaseException as e:
            errors.append(e)
            return 1

    f_c = N.NODE_EVALUATOR(node_eval)
    handles = (C.c_void_p * len(grids))(*[g.handle.value for g in grids])
    ls = np.ascontiguousarray(level_sums, dtype=np.int32)
    st = N.RefineStatsC()
    comm = _nccl_comm(dist) if (dist is not None and device) else None
    if comm is not None:
        import torch

        stream = torch.cuda.current_stream().cuda_stream
        status = N.lib.ddsg_refine_step_nccl(C.cast(handles, C.c_void_p), len(grids), ls.ctypes.data,
                                             C.cast(f_c, C.c_void_p), None, C.c_void_p(comm), rank, world,
                                             C.c_void_p(stream), C.byref(st))
        collective = "ncclAllGather over torch's communicator (native, device buffers)"
    else:
        ag_c = N.ALLGATHER_FN(allgather) if dist is not None else None
        status = N.lib.ddsg_refine_step(C.cast(handles, C.c_void_p), len(grids), ls.ctypes.data,
                                        C.cast(f_c, C.c_void_p), None, rank, world,
                                        C.cast(ag_c, C.c_void_p) if ag_c is not None else None, None,
                                        1 if device else 0, C.byref(st))
        collective = ("torch.distributed all-gather (%s)" % dist.get_backend()) if dist is not None else "none"
    if errors:
        raise errors[0]
    _check(status)
    for g in grids:  # max_level follows the appended level sums (ddsg_grid_append)
        lvl = C.c_int()
        _check(N.lib.ddsg_grid_info(g.handle, None, None, None, C.byref(lvl), None, None))
        g.max_level = lvl.value
    return RefineStats(new_nodes=st.new_nodes, rounds=st.rounds, gathered_bytes=st.gathered_bytes,
                       hierarchize_s=st.hierarchize_s, target_s=st.target_s, allgather_s=st.allgather_s,
                       collective=collective)
