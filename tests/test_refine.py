"""Refinement with the distributed all-gather on CPU:
one refinement step of config-5 component grids equals the reference-exact
build at the next level bit for bit, in one process and across 2 gloo ranks
(the grids stay identical on every rank)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import bits
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.refine import coords_of, refine_step

CFG = W.CONFIGS[5]
SLOTS = [((3,), 5, 6), ((17,), 5, 6), ((250,), 4, 5), ((3, 17), 3, 4), ((40, 299), 2, 3)]


def _grids(level_shift: int):
    return [W.build_cut_grid(CFG, dims, lo + level_shift, CFG.eps_1d if len(dims) == 1 else CFG.eps_2d)
            for dims, lo, hi in SLOTS]


def _f_eval():
    cuts = [W.CutTarget(CFG, dims) for dims, _, _ in SLOTS]
    return cuts, (lambda gi, xs: cuts[gi](xs))


def _level_sums():
    # refine from the top level sum of each grid: max_level + dim - 1
    return [lo + len(dims) - 1 for dims, lo, hi in SLOTS]


def test_coords_of_matches_reference_formula():
    keys = np.array([[1], [2], [3], [4], [7], [1 << 29]], dtype=np.uint32)
    want = [0.5, 0.25, 0.75, 0.125, 0.875, 2.0 ** -30]
    assert coords_of(keys)[:, 0].tolist() == want


def test_refine_step_single_process_equals_next_level_build():
    grids = _grids(0)
    cuts, f = _f_eval()
    stats = refine_step(grids, _level_sums(), f, dist=None, device=False)
    assert stats.new_nodes > 0
    direct = _grids(1)
    for g, h in zip(grids, direct):
        k1, s1 = g.nodes()
        k2, s2 = h.nodes()
        assert np.array_equal(k1, k2)
        assert np.array_equal(bits(s1), bits(s2))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grids = _grids(0)
        cuts, f = _f_eval()
        stats = refine_step(grids, _level_sums(), f, dist=dist, device=False)
        payload = {}
        for i, g in enumerate(grids):
            k, s = g.nodes()
            payload[f"k{i}"] = k
            payload[f"s{i}"] = s
        payload["gathered"] = np.array([stats.gathered_bytes])
        np.savez(f"{out_path}_{rank}.npz", **payload)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_refine_step_two_gloo_ranks(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path / "out")), nprocs=world, join=True)
    outs = [dict(np.load(tmp_path / f"out_{r}.npz")) for r in range(world)]
    direct = _grids(1)
    for i, h in enumerate(direct):
        k2, s2 = h.nodes()
        for o in outs:
            assert np.array_equal(o[f"k{i}"], k2)
            assert np.array_equal(bits(o[f"s{i}"]), bits(s2))
    assert outs[0]["gathered"][0] > 0


@pytest.mark.gpu
def test_refine_step_gpu_hierarchize_equals_next_level_build():
    """Same step with the new nodes hierarchized by the GPU kernels (EXACT,
    stored order): bit-identical to the reference-exact build at the next level."""
    grids = _grids(0)
    cuts, f = _f_eval()
    refine_step(grids, _level_sums(), f, dist=None, device=True)
    for g, h in zip(grids, _grids(1)):
        k1, s1 = g.nodes()
        k2, s2 = h.nodes()
        assert np.array_equal(k1, k2)
        assert np.array_equal(bits(s1), bits(s2))


def _config3_step(level: int, device: bool):
    """Config 3 (d = 20, adaptive, 2 stored-order runs at level 5) refined from
    `level` to `level + 1` by one refine_step: the reference's build caps the
    level sum at max_level + d - 1, so the next level is exactly one more
    batch (sparse_grid.hpp:84-108)."""
    import dataclasses

    lo = dataclasses.replace(W.CONFIGS[3], max_level=level)
    hi = dataclasses.replace(W.CONFIGS[3], max_level=level + 1)
    g = W.build_grid(lo)
    f = W.GridTarget(lo)
    stats = refine_step([g], [lo.max_level + lo.d - 1], lambda gi, xs: f(xs), dist=None, device=device)
    h = W.build_grid(hi)
    k1, s1 = g.nodes()
    k2, s2 = h.nodes()
    assert stats.new_nodes == h.size() - W.build_grid(lo).size() > 0
    assert np.array_equal(k1, k2)
    assert np.array_equal(bits(s1), bits(s2))


def test_refine_step_plain_grid_d20_host():
    _config3_step(3, device=False)


@pytest.mark.gpu
def test_refine_step_plain_grid_d20_gpu_hierarchize():
    _config3_step(4, device=True)


@pytest.mark.gpu
def test_hierarchize_device_rows_equal_host_rows():
    """ddsg_hierarchize with device f_values / surplus_out: the same bits as
    the host form (and as the reference's insert_batch on the host path)."""
    import torch

    grids = _grids(0)
    cuts, f = _f_eval()
    for gi, (g, s) in enumerate(zip(grids, _level_sums())):
        keys = g.refine_candidates(s)
        if len(keys) == 0:
            continue
        fv = f(gi, coords_of(keys))
        host = g.hierarchize(keys, fv, device=True)
        dev = g.hierarchize(keys, torch.from_numpy(fv).cuda()).cpu().numpy()
        ref = g.hierarchize(keys, fv, device=False)
        assert np.array_equal(bits(dev), bits(host)) and np.array_equal(bits(dev), bits(ref))
