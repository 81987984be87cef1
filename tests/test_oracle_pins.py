"""Pins the CPU oracle (oracle/ddsg_oracle.c) before it is trusted.

1. Known answers from the reference's own tests (restated, same inputs and
   thresholds): basis values (test_sparse_grid.cpp:31-41, 49-64), node counts
   (:66-75 with oracles.hpp:21-43), b coefficients (test_ddsg_eval.cpp:45-104).
2. The restatement against the reference itself (oracle/_ref, the unmodified
   headers compiled in place): bit-identical interpolate / evaluate_batch on
   plain, adaptive and HDMR grids, identical seeded points.
3. The golden fixtures under tests/golden/ (produced by the reference).
Runs on CPU.  Tests needing oracle/_ref skip when it was not built.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits, canonical_perm, golden_files, hdmr_slots_from_golden, int_ctx, load, wl

REF = O.ref() is not None
needs_ref = pytest.mark.skipif(not REF, reason="oracle/_ref not built (needs /root/reference)")


def basis(level, index, x, mode):
    return O.port().oracle_basis_value(mode, level, index, x)


# --------------------------------------------------------- known answers

def test_basis_known_answers():
    # test_sparse_grid.cpp:31-41
    assert basis(1, 1, 0.5, 0) == 1.0
    assert basis(2, 1, 0.5, 0) == 0.0
    assert abs(basis(2, 3, 0.6, 0) - 0.4) <= 1e-15
    assert basis(1, 1, 0.0, 1) == 1.0
    assert basis(2, 1, 0.0, 1) == 2.0
    assert basis(2, 3, 1.0, 1) == 2.0
    assert abs(basis(2, 3, 0.6, 1) - 0.4) <= 1e-15
    assert basis(3, 3, 0.375, 1) == 1.0


def test_basis_tensor_product_examples():
    # test_sparse_grid.cpp:49-64: basis_nd is the dim-ordered product
    assert basis(1, 1, 0.5, 0) * basis(1, 1, 0.5, 0) == 1.0
    assert basis(1, 1, 0.5, 0) * basis(2, 1, 0.0, 0) == 0.0
    assert abs(basis(2, 1, 0.25, 0) * basis(2, 3, 0.6, 0) - 0.4) <= 1e-15


@needs_ref
@pytest.mark.parametrize("level,index,x,mode", [
    (l, i, x, mode) for mode in (0, 1) for l in (1, 2, 3, 5, 12, 30) for i in (1, 3, (1 << l) - 1)
    if i <= (1 << l) - 1 and i % 2 == 1 for x in (0.0, 1.0, 0.3, 0.5, 2.0 ** -40, 1 - 2.0 ** -53, 0.123456789)
])
def test_basis_matches_reference_bitwise(level, index, x, mode):
    import ctypes as C

    out = C.c_double()
    assert O.ref().ref_basis_1d(level, index, x, mode, C.byref(out)) == 0
    assert bits(np.array([basis(level, index, x, mode)]))[0] == bits(np.array([out.value]))[0]


@needs_ref
def test_basis_rejects_invalid_pairs():
    import ctypes as C

    out = C.c_double()
    for l, i in ((2, 2), (2, 5), (0, 1)):  # test_sparse_grid.cpp:43-47
        assert O.ref().ref_basis_1d(l, i, 0.5, 0, C.byref(out)) == 1


def brute_node_count(n, L):
    """oracles.hpp:21-43 restated: all level vectors with |l|_1 <= L+n-1."""
    import itertools

    tot = 0
    for l in itertools.product(range(1, L + 1), repeat=n):
        if sum(l) <= L + n - 1:
            tot += 2 ** sum(v - 1 for v in l)
    return tot


@needs_ref
def test_node_counts_vs_reference_bruteforce():
    for n in range(1, 5):
        for L in range(1, 7):
            assert brute_node_count(n, L) == O.ref().ref_sg_node_count_bruteforce(n, L)


def test_b_coefficients_hand_derived():
    # test_ddsg_eval.cpp:45-73 via the oracle's subset-lattice walk
    import ctypes as C

    def b_of(family):
        order = np.array([len(u) for u in family], dtype=np.int32)
        dims = np.array([v for u in family for v in u] or [0], dtype=np.int32)
        out = np.zeros(len(family), dtype=np.int32)
        O.port().oracle_b_coefficients(len(family), order.ctypes.data, dims.ctypes.data, out.ctypes.data)
        return dict(zip(family, out.tolist()))

    assert b_of([(), (0,), (1,)]) == {(): -1, (0,): 1, (1,): 1}
    assert b_of([(), (0,), (1,), (2,)]) == {(): -2, (0,): 1, (1,): 1, (2,): 1}
    assert b_of([(), (0,), (1,), (0, 1)]) == {(): 0, (0,): 0, (1,): 0, (0, 1): 1}


@needs_ref
@pytest.mark.parametrize("d,k,eps_eta", [(d, k, e) for d in (2, 3, 4, 5) for k in range(1, min(3, d) + 1)
                                         for e in (0.0, 3e-3)])
def test_b_coefficients_match_reference_decompose(d, k, eps_eta):
    # test_ddsg_eval.cpp:75-104: families from real decompositions
    from paper_2202_06555_b200.workloads import telescoping_b

    keep, ctx = int_ctx(d)
    fn = "wl_coupled"
    fa, slots = O.ref_decompose(d, 1, k, 2, wl(fn), ctx, eps_eta=eps_eta)
    family = [s[0] for s in slots]
    want = [s[1] for s in slots]
    order = np.array([len(u) for u in family], dtype=np.int32)
    dims = np.array([v for u in family for v in u] or [0], dtype=np.int32)
    out = np.zeros(len(family), dtype=np.int32)
    O.port().oracle_b_coefficients(len(family), order.ctypes.data, dims.ctypes.data, out.ctypes.data)
    assert out.tolist() == want
    assert telescoping_b(family) == want


# ----------------------------------------------- restatement vs reference

@needs_ref
def test_uniform_points_match_reference_generator():
    from paper_2202_06555_b200.ddsg import uniform_points

    for seed, n, d in ((321, 1000, 8), (8443, 100, 4), (77001, 50, 2)):
        want = np.empty((n, d))
        O.ref().ref_uniform_points(d, n, seed, want.ctypes.data)
        assert np.array_equal(bits(O.port_uniform_points(seed, n, d)), bits(want))
        assert np.array_equal(bits(uniform_points(seed, n, d)), bits(want))


GRID_CASES = [
    ("wl_exp_product", 2, 1, 5, 0.0, 0, 2),
    ("wl_exp_product", 2, 1, 5, 0.0, 1, 2),
    ("wl_bump", 2, 1, 6, 1e-3, 1, None),
    ("wl_coupled", 5, 1, 4, 1e-3, 1, 5),
    ("wl_config1", 4, 1, 5, 0.0, 0, 4),
    ("wl_vector3", 2, 3, 5, 0.0, 1, None),
]


@needs_ref
@pytest.mark.parametrize("case", GRID_CASES, ids=lambda c: f"{c[0]}-d{c[1]}-mode{c[5]}")
def test_port_interpolate_matches_reference_bitwise(case):
    import ctypes as C

    fn, dim, m, L, eps, mode, cd = case
    keep, ctx = int_ctx(cd) if cd else (None, None)
    rc, g = O.ref_build(dim, m, mode, L, eps, wl(fn), C.c_void_p(ctx) if ctx else None)
    assert rc == 0
    keys, sur = g.nodes(dim, m)
    x = O.port_uniform_points(11 + dim, 2000, dim)
    x[:4] = np.array([0.0, 1.0, 0.5, 0.25])[:, None]
    rc, want = g.eval(x, m)
    assert rc == 0
    rc, got, bad = O.port_grid_eval(dim, m, mode, keys, sur, x)
    assert rc == 0
    assert np.array_equal(bits(got), bits(want))


@needs_ref
def test_port_hdmr_matches_reference_bitwise():
    # d=8, k=2, L=3 coupled (test_ddsg_eval.cpp:106-120 family), seed 321
    keep, ctx = int_ctx(8)
    fa, parts = O.ref_decompose(8, 1, 2, 3, wl("wl_coupled"), ctx)
    slots = [(u, b, (1, k, s) if k is not None else None) for u, b, k, s in parts]
    grids = [O.ref_from_nodes(len(u), 1, 1, 3, 0.0, k, s) if k is not None else None for u, b, k, s in parts]
    h = O.RefHdmr(8, 1, fa, [(u, b) for u, b, _, _ in parts], grids)
    x = O.port_uniform_points(321, 1000, 8)
    rc, want = h.eval(x, flat=False)
    assert rc == 0
    rc, got, _ = O.port_hdmr_eval(8, 1, fa, slots, x)
    assert rc == 0
    assert np.array_equal(bits(got), bits(want))
    rc, naive = h.eval_naive(x)
    assert np.max(np.abs(got - naive)) <= 1e-12  # vectorized == naive (test_ddsg_eval.cpp:119)


def test_port_domain_error_lowest_index():
    keys = np.array([[1, 1]], dtype=np.uint32)
    sur = np.array([[1.0]])
    x = np.full((10, 2), 0.5)
    x[7, 1] = 1.5
    x[4, 0] = np.nan
    rc, _, bad = O.port_grid_eval(2, 1, 0, keys, sur, x)
    assert rc == 2 and bad == 4


# ------------------------------------------------------------ golden files

@pytest.mark.parametrize("path", golden_files("grid"), ids=lambda p: p.stem)
def test_port_against_golden_grid(path):
    z = load(path)
    rc, y, _ = O.port_grid_eval(int(z["dim"]), int(z["m"]), int(z["mode"]), z["keys"], z["surplus"], z["x"])
    assert rc == 0
    assert np.array_equal(bits(y), bits(z["y_stored"]))
    p = canonical_perm(z["keys"])
    rc, yc, _ = O.port_grid_eval(int(z["dim"]), int(z["m"]), int(z["mode"]), z["keys"][p], z["surplus"][p], z["x"])
    assert np.array_equal(bits(yc), bits(z["y_canonical"]))


@pytest.mark.parametrize("path", golden_files("hdmr"), ids=lambda p: p.stem)
def test_port_against_golden_hdmr(path):
    z = load(path)
    for canonical, key in ((False, "y_stored"), (True, "y_canonical")):
        slots = hdmr_slots_from_golden(z, canonical=canonical)
        rc, y, _ = O.port_hdmr_eval(int(z["d"]), int(z["m"]), z["f_anchor"], slots, z["x"])
        assert rc == 0
        assert np.array_equal(bits(y), bits(z[key]))
