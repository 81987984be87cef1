"""GPU parity of the Morton-ordered plain-grid path (csrc/plain.cu): large
batches are sorted by a Morton key and each thread evaluates point perm[t].
It must be bit-identical to evaluation in input order and to the CPU
oracle, whatever the point order, batch size or domain errors."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits, canonical_perm, int_ctx, wl
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import (FAST, MODIFIED_LINEAR, ZERO_BOUNDARY, DomainError, SparseGridFunction,
                                        last_eval_stats, uniform_points)

pytestmark = pytest.mark.gpu


def _copy(g: SparseGridFunction, sort: bool, canonical: bool = False, sparse: bool = True) -> SparseGridFunction:
    """Same nodes (same order unless canonical), evaluated with (sort=True) or
    without the Morton pre-sort of the points, and for modified-linear grids
    on the sparse walk (sparse=True) or the dense walk."""
    keys, sur = g.nodes()
    if canonical:
        p = canonical_perm(keys)
        keys, sur = keys[p], sur[p]
    env = {"DDSG_PLAIN_SORT": "1" if sort else "0", "DDSG_PLAIN_SPARSE": "1" if sparse else "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        h = SparseGridFunction.from_nodes(g.dim, g.out_dim, g.max_level, g.eps_gamma, g.boundary_mode, keys, sur)
        h.interpolate(np.full((1, g.dim), 0.5))  # uploads the device program under these settings
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    return h


def _oracle(g: SparseGridFunction, x):
    keys, sur = g.nodes()
    rc, y, _ = O.port_grid_eval(g.dim, g.out_dim, g.boundary_mode, keys, sur, x)
    assert rc == 0
    return y


def _eval_sorted(g, x):
    y = g.interpolate(x)
    launches = last_eval_stats()[0]
    assert launches == 2, f"expected the sorted path (key kernel + evaluation kernel), got {launches} launches"
    return y


@pytest.fixture(scope="module")
def config2():
    return W.build_grid(W.CONFIGS[2])


@pytest.fixture(scope="module")
def config3():
    return W.build_grid(W.CONFIGS[3])


def test_config2_sorted_matches_direct_and_oracle(config2):
    cfg = W.CONFIGS[2]
    gt, gd = _copy(config2, True), _copy(config2, False)
    x = W.points(cfg, n=20000, seed=11)
    yt = _eval_sorted(gt, x)
    yd = gd.interpolate(x)
    assert last_eval_stats()[0] == 1
    assert np.array_equal(bits(yt), bits(yd))
    assert np.array_equal(bits(yt[:160]), bits(_oracle(config2, x[:160])))


@pytest.mark.parametrize("sparse", [True, False])
def test_config3_multirun_sorted_matches_direct_and_oracle(config3, sparse):
    """Config 3's adaptive build: 2 stored-order runs, partial subspaces,
    modified-linear boundary; sparse and dense walks, sorted and unsorted."""
    cfg = W.CONFIGS[3]
    gt, gd = _copy(config3, True, sparse=sparse), _copy(config3, False, sparse=not sparse)
    x = W.points(cfg, n=6000, seed=12)
    yt = _eval_sorted(gt, x)
    assert np.array_equal(bits(yt), bits(gd.interpolate(x)))
    assert np.array_equal(bits(yt[:96]), bits(_oracle(config3, x[:96])))


@pytest.mark.parametrize("m", [1, 5])
@pytest.mark.parametrize("mode", [ZERO_BOUNDARY, MODIFIED_LINEAR])
def test_sorted_edge_points(mode, m):
    """Cell boundaries, 0 and 1, repeated points (equal Morton keys), a batch
    that is not a multiple of the CTA size, both boundary modes, d = 7."""
    keep, ctx = int_ctx(7)
    g1 = SparseGridFunction.build(wl("wl_coupled"), 7, 1, 4, 1e-4, mode, ctx=ctx)
    keys, sur = g1.nodes()  # adaptive, stored order; m output columns
    sur_m = np.concatenate([sur * (1.0 + 0.1 * j) - 0.01 * j for j in range(m)], axis=1)
    g0 = SparseGridFunction.from_nodes(7, m, g1.max_level, g1.eps_gamma, mode, keys, sur_m)
    gt, gd = _copy(g0, True), _copy(g0, False, sparse=False)
    n = 5000 + 123
    x = uniform_points(321, n, 7)
    # dyadic cell boundaries, the ends, and subnormal / tiny coordinates (the
    # exponent-add scaling of factor() is exact for normal x and rounds away
    # exactly like 0 for subnormal x)
    edges = np.array([0.0, 1.0, 0.5, 0.25, 0.75, 0.125, 0.875, 1 - 2**-53, 2**-30, 2**-4,
                      5e-324, 1e-310, 2.0**-1022, 2**-60])
    rng = np.random.default_rng(5)
    x[:600] = edges[rng.integers(0, len(edges), size=(600, 7))]
    x[600:1200] = x[17]  # a whole tile's worth of one point
    x[1200:1300] = 0.5
    yt = _eval_sorted(gt, x)
    assert np.array_equal(bits(yt), bits(gd.interpolate(x)))
    sel = np.r_[0:600:7, 600:610, 1200:1210, n - 40:n]
    assert np.array_equal(bits(yt[sel]), bits(_oracle(g0, x[sel])))


def test_sorted_canonical_order():
    """Config 2's grid re-stored in canonical order (one run, same terms)."""
    cfg = W.CONFIGS[2]
    g2 = W.build_grid(cfg)
    gt = _copy(g2, True, canonical=True)
    gd = _copy(g2, False, canonical=True)
    x = W.points(cfg, n=8192, seed=99)
    yt = _eval_sorted(gt, x)
    assert np.array_equal(bits(yt), bits(gd.interpolate(x)))


def test_sorted_domain_error_lowest_index(config2):
    gt = _copy(config2, True)
    x = W.points(W.CONFIGS[2], n=9000, seed=3)
    x[7000, 4] = 1.0 + 1e-12
    x[4100, 9] = np.nan
    x[8000, 0] = -1e-300
    with pytest.raises(DomainError) as ei:
        gt.interpolate(x)
    assert ei.value.task_id == 4100


def test_sorted_fast_mode(config2):
    gt, gd = _copy(config2, True), _copy(config2, False)
    gt.set_eval_mode(FAST)
    gd.set_eval_mode(FAST)
    x = W.points(W.CONFIGS[2], n=8192, seed=4)
    assert np.array_equal(bits(_eval_sorted(gt, x)), bits(gd.interpolate(x)))


def test_sorted_device_buffers_and_permutation_invariance(config2):
    torch = pytest.importorskip("torch")
    gt = _copy(config2, True)
    x = W.points(W.CONFIGS[2], n=12000, seed=21)
    y = gt.interpolate(x)
    p = np.random.default_rng(2).permutation(len(x))
    xd = torch.from_numpy(x[p]).cuda()
    yd = torch.empty((len(x), config2.out_dim), dtype=torch.float64, device="cuda")
    gt.interpolate(xd, out=yd)
    assert np.array_equal(bits(yd.cpu().numpy()), bits(y[p]))


@pytest.mark.timeout(900)
def test_config3_level6_grid_exact():
    """Config 3's target refined to level 6 (1,262,721 nodes, 238 MB of
    surpluses; the reference's O(N^2) build cannot reach it, ours replays it
    in about 30 s): the Morton-sorted sparse walk against the oracle."""
    import dataclasses

    cfg = dataclasses.replace(W.CONFIGS[3], max_level=6)
    g = W.build_grid(cfg)
    assert g.size() == 1262721
    x = W.points(cfg, n=8192, seed=6)
    y = _eval_sorted(g, x)
    sel = np.r_[0:24, 8192 - 8:8192]
    assert np.array_equal(bits(y[sel]), bits(_oracle(g, x[sel])))


@pytest.mark.parametrize("dim", [24, 40])
def test_sparse_walk_beyond_20_dims(dim):
    """Modified-linear plain grids with 21..64 dims take the sparse walk (the
    dense walk stops at 20): against the generic kernel and the oracle."""
    keep, ctx = int_ctx(dim)
    g1 = SparseGridFunction.build(wl("wl_coupled"), dim, 1, 3, 1e-3, MODIFIED_LINEAR, ctx=ctx)
    keys, sur = g1.nodes()
    sur3 = np.concatenate([sur * (1.0 + 0.25 * j) for j in range(3)], axis=1)
    g0 = SparseGridFunction.from_nodes(dim, 3, g1.max_level, g1.eps_gamma, MODIFIED_LINEAR, keys, sur3)
    gs, gg = _copy(g0, True), _copy(g0, True, sparse=False)  # sparse walk / generic kernel
    x = uniform_points(77 + dim, 6000, dim)
    ys = _eval_sorted(gs, x)
    yg = gg.interpolate(x)
    assert last_eval_stats()[0] == 1  # the generic kernel, one launch
    assert np.array_equal(bits(ys), bits(yg))
    sel = np.r_[0:40, 5990:6000]
    assert np.array_equal(bits(ys[sel]), bits(_oracle(g0, x[sel])))
