"""Randomised parity: seeded random HDMR programs through every evaluation
path (slot kernel incl. order 3, multi-run carry, padded adaptive and
non-finite blocks, the generic kernel beyond the slot kernel's limits, the
small-batch path), bit for bit against the CPU oracle (the reference's
algorithm in stored node order) with the support hashes.

Each seed draws: d, m, a downward-closed family (all 1-d cuts, random pairs,
random triples with their pairs), per-order levels (some beyond the slot
kernel's static limits), random node subsets of the full grids (adaptive
blocks), random stored orders (several canonically sorted runs), the
boundary mode, telescoping or random coefficients b, occasional non-finite
surpluses, and batch sizes from 1 to a few thousand points with cell-boundary
and subnormal coordinates."""
from __future__ import annotations

import itertools
import json
import os
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits
from paper_2202_06555_b200.ddsg import MODIFIED_LINEAR, ZERO_BOUNDARY, SparseGridFunction, VectorizedDdsg
from paper_2202_06555_b200.workloads import telescoping_b

pytestmark = pytest.mark.gpu


def level_vectors(k: int, budget: int):
    """Level vectors l (l_j >= 1) with sum(l_j - 1) <= budget."""
    if k == 0:
        yield ()
        return
    for e in range(budget + 1):
        for rest in level_vectors(k - 1, budget - e):
            yield (e + 1,) + rest


def regular_keys(k: int, L: int) -> np.ndarray:
    """All nodes of the regular k-dim grid of level L (level sum <= L + k - 1)."""
    out = []
    for lv in level_vectors(k, L - 1):
        for cells in itertools.product(*[range(1 << (l - 1)) for l in lv]):
            out.append([(1 << (l - 1)) + c for l, c in zip(lv, cells)])
    return np.array(out, dtype=np.uint32).reshape(-1, k)


def random_program(seed: int):
    rng = np.random.default_rng(seed)
    d = int(rng.integers(3, 40))
    m = int(rng.choice([1, 3, 8, 9, 17, 33]))
    mode = int(rng.choice([ZERO_BOUNDARY, MODIFIED_LINEAR]))
    fam = {()} | {(j,) for j in range(d)}
    for _ in range(int(rng.integers(0, 12))):
        a, b = sorted(rng.choice(d, 2, replace=False).tolist())
        fam.add((a, b))
    if rng.random() < 0.4:
        for _ in range(int(rng.integers(1, 4))):
            t = tuple(sorted(rng.choice(d, 3, replace=False).tolist()))
            fam |= {t} | set(itertools.combinations(t, 2))
    fam = sorted(fam, key=lambda u: (len(u), u))
    levels = {1: int(rng.integers(1, 12)), 2: int(rng.integers(1, 8)), 3: int(rng.integers(1, 6))}
    b = telescoping_b(fam) if rng.random() < 0.7 else [int(v) for v in rng.integers(-3, 4, len(fam))]
    fa = rng.uniform(-2, 2, m)
    slots_o, slots_g = [], []
    for u, bu in zip(fam, b):
        if not u:
            slots_o.append((u, bu, None))
            slots_g.append((u, bu, None))
            continue
        k = len(u)
        L = levels[k]
        keys = regular_keys(k, L)
        if rng.random() < 0.5:  # adaptive: drop deep nodes at random
            lv = np.floor(np.log2(keys.astype(np.float64))).astype(int) + 1
            keep = (lv.sum(axis=1) <= k + 1) | (rng.random(len(keys)) < rng.uniform(0.3, 0.9))
            keys = keys[keep]
        if rng.random() < 0.3:  # stored order with several canonically sorted runs
            cut = int(rng.integers(1, len(keys))) if len(keys) > 1 else 0
            keys = np.concatenate([keys[cut:], keys[:cut]])
        sur = rng.uniform(-1, 1, (len(keys), m)) * 10.0 ** rng.uniform(-3, 3)
        if rng.random() < 0.05:
            sur[int(rng.integers(len(keys))), int(rng.integers(m))] = rng.choice([np.inf, -np.inf, np.nan])
        slots_o.append((u, bu, (mode, keys, sur)))
        slots_g.append((u, bu, SparseGridFunction.from_nodes(k, m, L, 0.0, mode, keys, sur)))
    vec = VectorizedDdsg.compile(d, m, fa, slots_g)
    n = int(rng.choice([1, 5, 256, 257, 1000, 3000]))
    x = O.port_uniform_points(seed, n, d)
    special = np.array([0.0, 1.0, 0.5, 0.25, 0.75, 1 - 2.0 ** -53, 2.0 ** -40, 5e-324])
    mask = rng.random(x.shape) < 0.05
    x[mask] = rng.choice(special, size=int(mask.sum()))
    return d, m, fa, slots_o, vec, x


@pytest.mark.parametrize("seed", range(200))
def test_random_program_bit_exact(seed):
    d, m, fa, slots_o, vec, x = random_program(seed)
    rc, want, _ = O.port_hdmr_eval(d, m, fa, slots_o, x)
    assert rc == 0
    y = vec.evaluate_batch(x)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(y), nan)
    assert np.array_equal(bits(y[~nan]), bits(want[~nan])), (
        f"seed {seed}: slot kernel {vec.uses_slot_kernel()}, {int((bits(y) != bits(want)).sum())} outputs differ")
    nnz_o, h_o = O.port_hdmr_support(d, m, slots_o, x)
    nnz, h = vec.support(x)
    assert np.array_equal(nnz, nnz_o) and np.array_equal(h, h_o)


def test_random_programs_cover_every_path():
    """The seeds above reach both the slot kernel and its fallback."""
    paths = {random_program(s)[4].uses_slot_kernel() for s in range(40)}
    assert paths == {True, False}


# ------------------------------------------------------------- plain grids

def random_grid(seed: int):
    """A random plain grid: d 1..24 (dense walk <= 20 dims, sparse walk for
    modified-linear grids up to 64, generic beyond), level 1..max for the
    dimension, random deep-node subsets, several stored-order runs, m 1..30,
    batches on both sides of the Morton-sort threshold (4096)."""
    rng = np.random.default_rng(10_000 + seed)
    d = int(rng.integers(1, 25))
    L = int(rng.integers(1, {1: 12, 2: 8, 3: 6}.get(d, 5 if d <= 8 else 3) + 1))
    m = int(rng.choice([1, 2, 5, 11, 21, 30]))
    mode = int(rng.choice([ZERO_BOUNDARY, MODIFIED_LINEAR]))
    keys = regular_keys(d, L)
    if rng.random() < 0.5:
        lv = np.floor(np.log2(keys.astype(np.float64))).astype(int) + 1
        keep = (lv.sum(axis=1) <= d + 1) | (rng.random(len(keys)) < rng.uniform(0.3, 0.9))
        keys = keys[keep]
    if rng.random() < 0.3 and len(keys) > 2:
        cut = int(rng.integers(1, len(keys)))
        keys = np.concatenate([keys[cut:], keys[:cut]])
    sur = rng.uniform(-1, 1, (len(keys), m)) * 10.0 ** rng.uniform(-3, 3)
    g = SparseGridFunction.from_nodes(d, m, L, 0.0, mode, keys, sur)
    n = int(rng.choice([1, 7, 300, 4096, 6000]))
    x = O.port_uniform_points(20_000 + seed, n, d)
    special = np.array([0.0, 1.0, 0.5, 0.125, 1 - 2.0 ** -53, 5e-324])
    mask = rng.random(x.shape) < 0.05
    x[mask] = rng.choice(special, size=int(mask.sum()))
    return d, m, mode, keys, sur, g, x


@pytest.mark.parametrize("seed", range(120))
def test_random_grid_bit_exact(seed):
    d, m, mode, keys, sur, g, x = random_grid(seed)
    rc, want, _ = O.port_grid_eval(d, m, mode, keys, sur, x)
    assert rc == 0
    y = g.interpolate(x)
    assert np.array_equal(bits(y), bits(want)), f"seed {seed}: {int((bits(y) != bits(want)).sum())} outputs differ"
    nnz_o, h_o = O.port_grid_support(d, mode, keys, x)
    nnz, h = g.support(x)
    assert np.array_equal(nnz, nnz_o) and np.array_equal(h, h_o)


# ------------------------------------------------------------------ campaign

@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("DDSG_CAMPAIGN") is None,
                    reason="long randomised campaign: set DDSG_CAMPAIGN=<seeds> (log in profiles/r2_parity_campaign.json)")
def test_random_campaign():
    """Seeds beyond the parametrised ones: DDSG_CAMPAIGN programs and as many
    plain grids, values and support hashes bit for bit; the summary goes to
    gpurun_out/parity_campaign.json."""
    count = int(os.environ["DDSG_CAMPAIGN"])
    bad, outputs, points, slot_kernel = [], 0, 0, 0
    for seed in range(1000, 1000 + count):
        d, m, fa, slots_o, vec, x = random_program(seed)
        rc, want, _ = O.port_hdmr_eval(d, m, fa, slots_o, x)
        y = vec.evaluate_batch(x)
        nan = np.isnan(want)
        nnz_o, h_o = O.port_hdmr_support(d, m, slots_o, x)
        nnz, h = vec.support(x)
        if rc != 0 or not (np.array_equal(np.isnan(y), nan) and np.array_equal(bits(y[~nan]), bits(want[~nan]))
                           and np.array_equal(nnz, nnz_o) and np.array_equal(h, h_o)):
            bad.append(("program", seed))
        outputs += y.size
        points += x.shape[0]
        slot_kernel += int(vec.uses_slot_kernel())
        d, m, mode, keys, sur, g, x = random_grid(seed)
        rc, want, _ = O.port_grid_eval(d, m, mode, keys, sur, x)
        y = g.interpolate(x)
        nnz_o, h_o = O.port_grid_support(d, mode, keys, x)
        nnz, h = g.support(x)
        if rc != 0 or not (np.array_equal(bits(y), bits(want)) and np.array_equal(nnz, nnz_o)
                           and np.array_equal(h, h_o)):
            bad.append(("grid", seed))
        outputs += y.size
        points += x.shape[0]
    out = Path(__file__).resolve().parent.parent / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / "parity_campaign.json").write_text(json.dumps({
        "what": "tests/test_gpu_random_programs.py::test_random_campaign: seeded random HDMR programs and plain grids "
                "(seeds 1000..), GPU values and support hashes against the CPU oracle, bit for bit",
        "programs": count, "grids": count, "programs_on_slot_kernel": slot_kernel, "points": points,
        "outputs": outputs, "mismatching_cases": bad}, indent=1))
    assert not bad, bad
