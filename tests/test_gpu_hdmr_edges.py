"""Edge cases of the HDMR evaluation path (slot kernel and its fallbacks),
each checked bit for bit against the CPU oracle on the same grid bits.

Grids are full grids with seeded random surpluses (the evaluation path does
not care how surpluses were obtained), so every case is cheap to set up."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits
from paper_2202_06555_b200.ddsg import (MODIFIED_LINEAR, ZERO_BOUNDARY, SparseGridFunction, VectorizedDdsg,
                                        uniform_points)
from paper_2202_06555_b200.workloads import telescoping_b

pytestmark = pytest.mark.gpu


def full_keys(k: int, L: int) -> np.ndarray:
    """All nodes of the regular k-dim grid of level L in canonical order."""
    out = []
    for s in range(k, L + k):
        for lv in itertools.product(range(1, L + 1), repeat=k):
            if sum(lv) != s:
                continue
            for cells in itertools.product(*[range(1 << (l - 1)) for l in lv]):
                out.append([(1 << (l - 1)) + c for l, c in zip(lv, cells)])
    return np.array(sorted(out, key=lambda key: (sum(int(v).bit_length() for v in key), key)), dtype=np.uint32)


def make(d, m, family, levels, mode=MODIFIED_LINEAR, b=None, seed=0, poison=None):
    rng = np.random.default_rng(seed)
    b = telescoping_b(family) if b is None else b
    slots_o, slots_g = [], []
    fa = rng.uniform(-1, 1, m)
    for u, bu in zip(family, b):
        if not u:
            slots_o.append((u, bu, None))
            slots_g.append((u, bu, None))
            continue
        keys = full_keys(len(u), levels[len(u)])
        sur = rng.uniform(-1, 1, (len(keys), m))
        if poison is not None and u == poison[0]:
            sur[poison[1] % len(keys), poison[2] % m] = poison[3]
        slots_o.append((u, bu, (mode, keys, sur)))
        slots_g.append((u, bu, SparseGridFunction.from_nodes(len(u), m, levels[len(u)], 0.0, mode, keys, sur)))
    vec = VectorizedDdsg.compile(d, m, fa, slots_g)
    return vec, fa, slots_o


def check(vec, d, m, fa, slots_o, x, nan_ok=False):
    rc, want, _ = O.port_hdmr_eval(d, m, fa, slots_o, x)
    assert rc == 0
    y = vec.evaluate_batch(x)
    if nan_ok:
        assert np.array_equal(np.isnan(y), np.isnan(want))
        mask = ~np.isnan(want)
        assert np.array_equal(bits(y[mask]), bits(want[mask]))
    else:
        assert np.array_equal(bits(y), bits(want))
    nnz_o, h_o = O.port_hdmr_support(d, m, slots_o, x)
    nnz, h = vec.support(x)
    assert np.array_equal(nnz, nnz_o) and np.array_equal(h, h_o)


def pts(d, n=700, seed=5):
    x = uniform_points(seed, n, d)
    x[:6] = np.array([0.0, 1.0, 0.5, 0.25, 1 - 2.0 ** -53, 2.0 ** -40])[:, None]
    x[6:9] = np.array([5e-324, 1e-310, 2.0 ** -1022])[:, None]  # subnormal / smallest normal coordinates
    return x


def family_1d_2d(d, pairs):
    return [()] + [(j,) for j in range(d)] + sorted(pairs)


def test_only_anchor_slot():
    d, m = 3, 5
    vec, fa, so = make(d, m, [()], {})
    check(vec, d, m, fa, so, pts(d))


def test_empty_batch():
    vec, fa, so = make(4, 3, family_1d_2d(4, [(0, 1)]), {1: 4, 2: 3})
    assert vec.evaluate_batch(np.zeros((0, 4))).shape == (0, 3)


@pytest.mark.parametrize("mode", [ZERO_BOUNDARY, MODIFIED_LINEAR])
@pytest.mark.parametrize("m", [1, 8, 9, 23])
def test_modes_and_column_blocks(mode, m):
    d = 6
    fam = family_1d_2d(d, [(0, 1), (1, 2), (2, 5), (3, 4)])
    vec, fa, so = make(d, m, fam, {1: 6, 2: 4}, mode=mode, seed=m)
    assert vec.uses_slot_kernel()
    check(vec, d, m, fa, so, pts(d))


def test_b_kinds():
    # b = 1, -1, 2 (power of two), -3 (general DMUL), 0 (skipped)
    d, m = 4, 7
    fam = family_1d_2d(d, [(0, 1), (2, 3)])
    b = [5, 1, -1, 2, -3, 1, 0]
    vec, fa, so = make(d, m, fam, {1: 5, 2: 3}, b=b)
    check(vec, d, m, fa, so, pts(d))


def test_non_finite_surplus_takes_general_path():
    d, m = 4, 3
    fam = family_1d_2d(d, [(0, 1)])
    vec, fa, so = make(d, m, fam, {1: 5, 2: 3}, poison=((0, 1), 7, 1, np.inf))
    check(vec, d, m, fa, so, pts(d), nan_ok=True)


@pytest.mark.parametrize("L1,expect_slot_kernel", [(10, True), (11, False)])
def test_deep_1d_cuts(L1, expect_slot_kernel):
    d, m = 3, 9
    fam = family_1d_2d(d, [(0, 2)])
    vec, fa, so = make(d, m, fam, {1: L1, 2: 4})
    assert vec.uses_slot_kernel() == expect_slot_kernel
    check(vec, d, m, fa, so, pts(d, 400))


@pytest.mark.parametrize("mode", [ZERO_BOUNDARY, MODIFIED_LINEAR])
@pytest.mark.parametrize("L3", [1, 2, 3, 4])
def test_order3_slots_on_the_slot_kernel(mode, L3):
    """k_max = 3 families (decompose supports them, hdmr.hpp:364): order-3
    slots with level sums <= 6 run on the slot kernel (leaf_full3), bit-exact."""
    d, m = 6, 9
    fam = ([()] + [(j,) for j in range(d)] + [(0, 1), (0, 2), (1, 2), (2, 4), (3, 5)]
           + [(0, 1, 2)])
    vec, fa, so = make(d, m, fam, {1: 5, 2: 4, 3: L3}, mode=mode, seed=L3)
    assert vec.uses_slot_kernel()
    check(vec, d, m, fa, so, pts(d, 500))


def _partial_triple(m, rng, drop, poison=False):
    keys = full_keys(3, 4)
    lv = np.floor(np.log2(keys.astype(np.float64))).astype(int) + 1
    deep = lv.sum(axis=1) >= 5
    keep = ~(deep & (rng.random(len(keys)) < drop))
    keys = keys[keep]
    sur = rng.uniform(-1, 1, (len(keys), m))
    if poison:
        sur[len(keys) // 2, 1] = np.inf
    return keys, sur


@pytest.mark.parametrize("poison", [False, True])
def test_order3_adaptive_slots(poison):
    """Partial order-3 grids: padded to the full grid (finite surpluses) or
    walked through the slab (non-finite surpluses), bit-exact."""
    rng = np.random.default_rng(5)
    d, m = 4, 7
    family = [(), (0,), (1,), (2,), (3,), (0, 1), (0, 2), (1, 2), (0, 1, 2)]
    b = telescoping_b(family)
    fa = rng.uniform(-1, 1, m)
    slots_o, slots_g = [], []
    for u, bu in zip(family, b):
        if not u:
            slots_o.append((u, bu, None))
            slots_g.append((u, bu, None))
            continue
        if len(u) == 3:
            keys, sur = _partial_triple(m, rng, 0.4, poison)
        else:
            keys = full_keys(len(u), 4)
            sur = rng.uniform(-1, 1, (len(keys), m))
        slots_o.append((u, bu, (MODIFIED_LINEAR, keys, sur)))
        slots_g.append((u, bu, SparseGridFunction.from_nodes(len(u), m, 4, 0.0, MODIFIED_LINEAR, keys, sur)))
    vec = VectorizedDdsg.compile(d, m, fa, slots_g)
    assert vec.uses_slot_kernel()
    check(vec, d, m, fa, slots_o, pts(d, 600), nan_ok=poison)


@pytest.mark.parametrize("levels,k", [({1: 4, 2: 3, 3: 5}, 3), ({1: 3, 2: 3, 3: 2, 4: 2}, 4)])
def test_beyond_the_slot_kernel_falls_back_exactly(levels, k):
    """Order-3 slots of level sum > 6 and order-4 slots run on the generic
    kernel, still bit-exact."""
    d, m = 5, 5
    fam = [()] + [(j,) for j in range(d)] + [(0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (2, 3)] + [(0, 1, 2)]
    if k == 4:
        fam += [(0, 1, 3), (0, 2, 3), (1, 2, 3), (0, 1, 2, 3)]
    fam = sorted(fam, key=lambda u: (len(u), u))
    vec, fa, so = make(d, m, fam, levels)
    assert not vec.uses_slot_kernel()
    check(vec, d, m, fa, so, pts(d, 300))


def test_many_slots_deep_tree():
    # 1 + 60 + 200 slots -> 9 tree levels (TMEM + shared-memory levels)
    d, m = 60, 3
    rng = np.random.default_rng(1)
    pairs = set()
    while len(pairs) < 200:
        a, b = sorted(rng.choice(d, 2, replace=False).tolist())
        pairs.add((a, b))
    fam = family_1d_2d(d, pairs)
    vec, fa, so = make(d, m, fam, {1: 3, 2: 2})
    assert vec.uses_slot_kernel()
    check(vec, d, m, fa, so, pts(d, 600))


@pytest.mark.parametrize("mode", [MODIFIED_LINEAR, ZERO_BOUNDARY])
def test_order2_subspace_beyond_max_single_level(mode):
    """A pair grid holding (2,2) but no level-3 subspace: its max single level
    is 2 while its level sum reaches 4, so the slot kernel must walk every
    (l1, l2) with l1 + l2 <= 4 (nlev = max level sum - 1)."""
    rng = np.random.default_rng(11)
    keys = [k for k in full_keys(2, 3) if all(int(v).bit_length() <= 2 for v in k)]
    keys = np.array(keys, dtype=np.uint32)
    assert any(int(a).bit_length() == 2 and int(b).bit_length() == 2 for a, b in keys)
    d, m = 3, 5
    family = [(), (0,), (1,), (2,), (0, 2)]
    b = telescoping_b(family)
    fa = rng.uniform(-1, 1, m)
    slots_o, slots_g = [], []
    for u, bu in zip(family, b):
        if not u:
            slots_o.append((u, bu, None))
            slots_g.append((u, bu, None))
            continue
        kk = keys if len(u) == 2 else full_keys(1, 4)
        sur = rng.uniform(-1, 1, (len(kk), m))
        slots_o.append((u, bu, (mode, kk, sur)))
        slots_g.append((u, bu, SparseGridFunction.from_nodes(len(u), m, 4, 0.0, mode, kk, sur)))
    vec = VectorizedDdsg.compile(d, m, fa, slots_g)
    assert vec.uses_slot_kernel()
    check(vec, d, m, fa, slots_o, pts(d))


def test_programs_with_different_stage_sizes_coexist():
    """The slot kernel's dynamic shared-memory limit belongs to the kernel
    function, not the program: a program with large stages must still launch
    after a program with small stages was built (and vice versa)."""
    d, m = 3, 9
    big, fa_b, so_b = make(d, m, family_1d_2d(d, [(0, 2)]), {1: 10, 2: 4}, seed=1)
    small, fa_s, so_s = make(d, m, family_1d_2d(d, []), {1: 2, 2: 2}, seed=2)
    assert big.uses_slot_kernel() and small.uses_slot_kernel()
    check(big, d, m, fa_b, so_b, pts(d, 300))
    check(small, d, m, fa_s, so_s, pts(d, 300))
    check(big, d, m, fa_b, so_b, pts(d, 300, seed=9))


def test_concurrent_programs_on_host_threads():
    """Two programs with different stage sizes evaluated concurrently from
    two host threads (per-thread scratch and streams; the shared-memory limit
    of the shared kernel is only ever raised): every result stays bit-identical
    to its single-threaded evaluation."""
    import threading

    d, m = 3, 9
    big, fa_b, so_b = make(d, m, family_1d_2d(d, [(0, 2)]), {1: 10, 2: 4}, seed=3)
    small, fa_s, so_s = make(d, m, family_1d_2d(d, [(1, 2)]), {1: 3, 2: 2}, seed=4)
    xb, xs = pts(d, 5000, seed=11), pts(d, 5000, seed=12)
    want_b, want_s = bits(big.evaluate_batch(xb)), bits(small.evaluate_batch(xs))
    errors = []

    def run(vec, x, want):
        try:
            for _ in range(20):
                if not np.array_equal(bits(vec.evaluate_batch(x)), want):
                    errors.append("mismatch")
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    ts = [threading.Thread(target=run, args=a) for a in ((big, xb, want_b), (small, xs, want_s))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:3]


# ------------------------------------------------ small batches (n <= 256)
# Few points take the slot-parallel path (one thread per point x slot x
# column chunk, then the pairwise tree per point, height by height): the
# per-point evaluate(x, out, ws) of the reference's callers.

@pytest.mark.parametrize("n", [1, 2, 7, 256, 257])
@pytest.mark.parametrize("case", ["modes", "b_kinds", "nonfinite", "deep_tree", "order3"])
def test_small_batches_bit_exact(case, n):
    if case == "modes":
        d, m = 6, 23
        vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1), (1, 2), (2, 5), (3, 4)]), {1: 6, 2: 4},
                           mode=ZERO_BOUNDARY, seed=n)
    elif case == "b_kinds":
        d, m = 4, 7
        vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1), (2, 3)]), {1: 5, 2: 3}, b=[5, 1, -1, 2, -3, 1, 0])
    elif case == "nonfinite":
        d, m = 4, 3
        vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1)]), {1: 5, 2: 3}, poison=((0, 1), 7, 1, np.inf))
    elif case == "deep_tree":
        d, m = 60, 3
        rng = np.random.default_rng(1)
        pairs = set()
        while len(pairs) < 200:
            a, b = sorted(rng.choice(d, 2, replace=False).tolist())
            pairs.add((a, b))
        vec, fa, so = make(d, m, family_1d_2d(d, pairs), {1: 3, 2: 2})
    else:
        d, m = 4, 5
        fam = [()] + [(j,) for j in range(d)] + [(0, 1), (0, 2), (1, 2)] + [(0, 1, 2)]
        vec, fa, so = make(d, m, fam, {1: 4, 2: 3, 3: 5})  # order 3 beyond the slot kernel
    check(vec, d, m, fa, so, pts(d, max(n, 9))[:n], nan_ok=case == "nonfinite")


def test_small_batch_domain_error_lowest_index():
    from paper_2202_06555_b200.ddsg import DomainError

    d, m = 4, 5
    vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1)]), {1: 4, 2: 3})
    x = pts(d, 9)
    x[5, 2] = np.nan
    x[7, 0] = 1.5
    with pytest.raises(DomainError) as e:
        vec.evaluate_batch(x)
    assert e.value.task_id == 5


# ------------------------------------- mid-size batches (a few point tiles)
# Fewer CTAs than SMs: the pairwise tree is cut at depth S and its 2^S
# subtrees run as concurrent launches over their own block ranges, the
# subtree roots added in tree order (fast_hdmr.cuh).  Same leaves, same
# merges: bit-identical, checked against the oracle; the launch count shows
# the split was taken.

@pytest.mark.parametrize("n", [257, 300, 513, 1300, 2100])
@pytest.mark.parametrize("case", ["modes", "b_kinds", "nonfinite", "deep_tree", "order3", "wide"])
def test_mid_batches_split_bit_exact(case, n):
    from paper_2202_06555_b200.ddsg import last_eval_stats

    if case == "modes":
        d, m = 6, 23
        vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1), (1, 2), (2, 5), (3, 4)]), {1: 6, 2: 4},
                           mode=ZERO_BOUNDARY, seed=n)
    elif case == "b_kinds":
        d, m = 4, 7
        vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1), (2, 3)]), {1: 5, 2: 3}, b=[5, 1, -1, 2, -3, 1, 0])
    elif case == "nonfinite":
        d, m = 4, 3
        vec, fa, so = make(d, m, family_1d_2d(d, [(0, 1)]), {1: 5, 2: 3}, poison=((0, 1), 7, 1, np.inf))
    elif case == "deep_tree":
        d, m = 60, 3
        rng = np.random.default_rng(1)
        pairs = set()
        while len(pairs) < 200:
            a, b = sorted(rng.choice(d, 2, replace=False).tolist())
            pairs.add((a, b))
        vec, fa, so = make(d, m, family_1d_2d(d, pairs), {1: 3, 2: 2})
    elif case == "order3":
        d, m = 5, 9
        fam = [()] + [(j,) for j in range(d)] + [(0, 1), (0, 2), (1, 2), (3, 4)] + [(0, 1, 2)]
        vec, fa, so = make(d, m, fam, {1: 5, 2: 3, 3: 3})
    else:  # many slots and many column blocks: the split depth shrinks with the CTA count
        d, m = 40, 70
        vec, fa, so = make(d, m, family_1d_2d(d, [(j, j + 1) for j in range(0, 40, 2)] + [(0, 39), (5, 30)]),
                           {1: 4, 2: 3})
    assert vec.uses_slot_kernel()
    x = pts(d, n, seed=n)
    check(vec, d, m, fa, so, x, nan_ok=case == "nonfinite")
    vec.evaluate_batch(x)
    launches = last_eval_stats()[0]
    tiles, n_cb = -(-n // 512), -(-m // 8)
    if tiles * n_cb * 2 <= 148 and len(so) >= 64:  # (few slots: one launch is cheaper than the fork/join)
        assert launches > 2, (launches, tiles, n_cb)  # transpose + 2^S subtrees + combine


# The small-batch forms (fused one-launch kernel / rows + tree kernels) and the
# split launches are chosen by switches read once per process: run a few
# programs in child processes under each setting and compare the raw bits.

_CHILD = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np
from test_gpu_random_programs import random_program
from helpers import bits
h = hashlib.sha256()
for seed in (3, 11, 42, 77):
    d, m, fa, slots_o, vec, x = random_program(seed)
    for n in (1, 5, 40, 300):
        xs = np.ascontiguousarray(np.resize(x, (n, d)))
        h.update(bits(vec.evaluate_batch(xs)).tobytes())
print(h.hexdigest())
"""


def test_small_and_mid_batch_forms_agree_bitwise():
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    digests = {}
    for name, env in {"default": {}, "fused_everywhere": {"DDSG_SMALL_FUSED": "2"},
                      "two_kernels": {"DDSG_SMALL_FUSED": "0"}, "slot_rows": {"DDSG_SMALL_FUSED": "0", "DDSG_SMALL_TERMS": "0"},
                      "no_split": {"DDSG_SLOT_SPLIT": "0"},
                      "slot_kernel_only": {"DDSG_SMALL_BATCH": "0"}}.items():
        out = subprocess.run([sys.executable, "-c", _CHILD, root], env={**os.environ, **env}, capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        digests[name] = out.stdout.strip().splitlines()[-1]
    assert len(set(digests.values())) == 1, digests
