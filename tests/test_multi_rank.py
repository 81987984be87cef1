"""Multi-rank paths: points shard with no data-path
collective, grids are built once and broadcast, and the only collective is
the refinement all-gather.

CPU (gloo, 2 ranks): the broadcast of rank 0's grids reproduces the local
build bit for bit on every rank.
GPU: two processes on the one GPU (gloo for the host-side gather; their
kernels never wait on each other) evaluate contiguous shards of ONE seeded
point set: the concatenation is bitwise the 1-process evaluation.  And the
native refinement step over torch's NCCL communicator (a one-rank group:
NCCL refuses two ranks on one device) equals the next-level build."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import bits
from paper_2202_06555_b200 import workloads as W

BLOCK = 1 << 14


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port, backend):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def _bcast_worker(rank, world, port, out_path):
    dist = _init(rank, world, port, "gloo")
    try:
        parts = W.broadcast_hdmr_parts(W.CONFIGS[4], dist, "cpu")
        payload = {}
        for i, (u, b, g) in enumerate(parts.slots):
            if g is not None:
                k, s = g.nodes()
                payload[f"k{i}"], payload[f"s{i}"] = k, s
                payload[f"l{i}"] = np.array([g.max_level])
        payload["fa"] = parts.f_anchor
        np.savez(f"{out_path}_{rank}.npz", **payload)
    finally:
        dist.destroy_process_group()


def test_build_once_broadcast_equals_local_build(tmp_path):
    world = 2
    mp.spawn(_bcast_worker, args=(world, _free_port(), str(tmp_path / "b")), nprocs=world, join=True)
    local = W.build_hdmr_parts(W.CONFIGS[4])
    outs = [dict(np.load(tmp_path / f"b_{r}.npz")) for r in range(world)]
    for o in outs:
        assert np.array_equal(bits(o["fa"]), bits(local.f_anchor))
        for i, (u, b, g) in enumerate(local.slots):
            if g is None:
                continue
            k, s = g.nodes()
            assert np.array_equal(o[f"k{i}"], k) and np.array_equal(bits(o[f"s{i}"]), bits(s))
            assert int(o[f"l{i}"][0]) == g.max_level


def _shard_worker(rank, world, port, n_total, out_path):
    import torch

    from paper_2202_06555_b200.ddsg import uniform_point_blocks

    dist = _init(rank, world, port, "gloo")
    try:
        torch.cuda.set_device(0)
        cfg = W.CONFIGS[4]
        parts = W.broadcast_hdmr_parts(cfg, dist, "cpu")
        from paper_2202_06555_b200.ddsg import VectorizedDdsg

        vec = VectorizedDdsg.compile(parts.d, parts.m, parts.f_anchor, parts.slots)
        n_local = n_total // world
        first = rank * n_local
        x = torch.from_numpy(uniform_point_blocks(cfg.seed, BLOCK, first, n_local, cfg.d)).cuda()
        y = vec.evaluate_batch(x).cpu().numpy()
        np.save(f"{out_path}_{rank}.npy", y)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2])
def test_sharded_evaluation_is_bitwise_the_one_rank_evaluation(tmp_path, world):
    """outputs are bitwise independent of the rank count."""
    import torch

    from paper_2202_06555_b200.ddsg import uniform_point_blocks

    n_total = 3 * BLOCK + 1000 * world  # shard boundaries inside a point block
    mp.spawn(_shard_worker, args=(world, _free_port(), n_total, str(tmp_path / "y")), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"y_{r}.npy") for r in range(world)])
    cfg = W.CONFIGS[4]
    vec = W.build_hdmr(cfg)[0]
    x = torch.from_numpy(uniform_point_blocks(cfg.seed, BLOCK, 0, n_total, cfg.d)).cuda()
    want = vec.evaluate_batch(x).cpu().numpy()
    assert got.shape == want.shape
    assert np.array_equal(bits(got), bits(want))


def _nccl_refine_worker(rank, world, port, out_path):
    import torch

    from paper_2202_06555_b200.refine import refine_step

    torch.cuda.set_device(0)
    dist = _init(rank, world, port, "nccl")
    try:
        cfg = W.CONFIGS[5]
        slots = [((3,), 5), ((250,), 4), ((3, 17), 3)]
        grids = [W.build_cut_grid(cfg, u, lvl, cfg.eps_1d if len(u) == 1 else cfg.eps_2d) for u, lvl in slots]
        cuts = [W.CutTarget(cfg, u) for u, _ in slots]
        st = refine_step(grids, [lvl + len(u) - 1 for u, lvl in slots], lambda gi, xs: cuts[gi](xs), dist=dist,
                         device=True)
        payload = {"new": np.array([st.new_nodes]), "gathered": np.array([st.gathered_bytes]),
                   "nccl": np.array([int("nccl" in st.collective.lower())])}
        for i, g in enumerate(grids):
            k, s = g.nodes()
            payload[f"k{i}"], payload[f"s{i}"] = k, s
        np.savez(f"{out_path}_{rank}.npz", **payload)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_native_refinement_over_torch_nccl_communicator(tmp_path):
    """ddsg_refine_step_nccl with torch's ncclComm_t (one-rank group): the
    all-gather runs (device buffers, ncclAllGather) and the refined grids
    equal the reference-exact build at the next level."""
    mp.spawn(_nccl_refine_worker, args=(1, _free_port(), str(tmp_path / "r")), nprocs=1, join=True)
    o = dict(np.load(tmp_path / "r_0.npz"))
    assert o["new"][0] > 0 and o["gathered"][0] > 0 and o["nccl"][0] == 1
    cfg = W.CONFIGS[5]
    for i, (u, lvl) in enumerate([((3,), 5), ((250,), 4), ((3, 17), 3)]):
        h = W.build_cut_grid(cfg, u, lvl + 1, cfg.eps_1d if len(u) == 1 else cfg.eps_2d)
        k, s = h.nodes()
        assert np.array_equal(o[f"k{i}"], k) and np.array_equal(bits(o[f"s{i}"]), bits(s))


def _gloo_device_refine_worker(rank, world, port, out_path):
    import torch

    from paper_2202_06555_b200.refine import refine_step

    torch.cuda.set_device(0)
    dist = _init(rank, world, port, "gloo")
    try:
        cfg = W.CONFIGS[5]
        slots = [((3,), 5), ((250,), 4), ((3, 17), 3), ((40, 299), 2)]
        grids = [W.build_cut_grid(cfg, u, lvl, cfg.eps_1d if len(u) == 1 else cfg.eps_2d) for u, lvl in slots]
        cuts = [W.CutTarget(cfg, u) for u, _ in slots]
        st = refine_step(grids, [lvl + len(u) - 1 for u, lvl in slots], lambda gi, xs: cuts[gi](xs), dist=dist,
                         device=True)
        payload = {"new": np.array([st.new_nodes]), "gathered": np.array([st.gathered_bytes])}
        for i, g in enumerate(grids):
            k, s = g.nodes()
            payload[f"k{i}"], payload[f"s{i}"] = k, s
        np.savez(f"{out_path}_{rank}.npz", **payload)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_native_refinement_two_ranks_device_rows(tmp_path):
    """ddsg_refine_step with two ranks on the one GPU: each hierarchizes its
    share into device rows, the all-gather callback (gloo) exchanges them,
    both ranks append identically -- the reference-exact next-level build."""
    world = 2
    mp.spawn(_gloo_device_refine_worker, args=(world, _free_port(), str(tmp_path / "g")), nprocs=world, join=True)
    outs = [dict(np.load(tmp_path / f"g_{r}.npz")) for r in range(world)]
    cfg = W.CONFIGS[5]
    assert outs[0]["new"][0] > 0 and outs[0]["gathered"][0] > 0
    for i, (u, lvl) in enumerate([((3,), 5), ((250,), 4), ((3, 17), 3), ((40, 299), 2)]):
        h = W.build_cut_grid(cfg, u, lvl + 1, cfg.eps_1d if len(u) == 1 else cfg.eps_2d)
        k, s = h.nodes()
        for o in outs:
            assert np.array_equal(o[f"k{i}"], k) and np.array_equal(bits(o[f"s{i}"]), bits(s))
