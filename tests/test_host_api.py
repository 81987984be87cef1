"""Host side of the drop-in boundary (CPU only, no kernel launches):
the C-ABI library loads and exports every symbol include/ddsg_b200.h
declares; grid construction reproduces the reference's build bit for bit;
argument validation follows the reference's exception contract."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits, int_ctx, wl
from paper_2202_06555_b200 import _native as N
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import (MODIFIED_LINEAR, ZERO_BOUNDARY, BuildError, InvalidArgument,
                                        SparseGridFunction, VectorizedDdsg)

ROOT = Path(__file__).resolve().parent.parent
REF = O.ref() is not None
needs_ref = pytest.mark.skipif(not REF, reason="oracle/_ref not built (needs /root/reference)")


def header_functions():
    text = (ROOT / "include" / "ddsg_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ddsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(N.lib, n)]
    assert not missing, missing
    assert set(N.SIGNATURES) >= set(names)


def test_library_has_device_kernels_for_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


# ------------------------------------------------------------ grid build

BUILD_CASES = [
    ("wl_exp_product", 2, 1, 5, 0.0, ZERO_BOUNDARY, 2),
    ("wl_exp_product", 2, 1, 5, 0.0, MODIFIED_LINEAR, 2),
    ("wl_bump", 2, 1, 6, 1e-3, MODIFIED_LINEAR, None),
    ("wl_coupled", 3, 1, 6, 1e-4, MODIFIED_LINEAR, 3),
    ("wl_coupled", 4, 1, 5, 1e-3, ZERO_BOUNDARY, 4),
    ("wl_config1", 4, 1, 5, 0.0, ZERO_BOUNDARY, 4),
    ("wl_vector3", 2, 3, 6, 1e-3, MODIFIED_LINEAR, None),
    ("wl_config3", 20, 21, 3, 1e-3, MODIFIED_LINEAR, None),
]


@needs_ref
@pytest.mark.parametrize("case", BUILD_CASES, ids=lambda c: f"{c[0]}-d{c[1]}-L{c[3]}-eps{c[4]}-mode{c[5]}")
def test_build_matches_reference_bitwise(case):
    """SparseGridFunction::build (sparse_grid.hpp:84-108): same node set, same
    stored order, same surplus bits, same quadrature."""
    fn, dim, m, L, eps, mode, cd = case
    keep, ctx = int_ctx(cd) if cd else (None, 0)
    g = SparseGridFunction.build(wl(fn), dim, m, L, eps, mode, ctx=ctx)
    rc, rg = O.ref_build(dim, m, mode, L, eps, wl(fn), C.c_void_p(ctx) if ctx else None)
    assert rc == 0
    k1, s1 = g.nodes()
    k2, s2 = rg.nodes(dim, m)
    assert np.array_equal(k1, k2)
    assert np.array_equal(bits(s1), bits(s2))
    assert np.array_equal(bits(g.quadrature()), bits(rg.quadrature(m)))


def test_node_counts_match_bruteforce():
    # test_sparse_grid.cpp:66-75
    import itertools

    def brute(n, L):
        return sum(2 ** sum(v - 1 for v in l) for l in itertools.product(range(1, L + 1), repeat=n)
                   if sum(l) <= L + n - 1)

    f = wl("wl_constant")
    assert SparseGridFunction.build(f, 1, 1, 3, 0.0, ZERO_BOUNDARY).size() == 7
    assert SparseGridFunction.build(f, 2, 1, 2, 0.0, ZERO_BOUNDARY).size() == 5
    for n in range(1, 5):
        for L in range(1, 7):
            assert SparseGridFunction.build(f, n, 1, L, 0.0, MODIFIED_LINEAR).size() == brute(n, L)


def test_single_basis_target_stops_refining():
    # test_sparse_grid.cpp:77-86
    hat = lambda x: np.maximum(1.0 - 2.0 * np.abs(x[:, 0] - 0.5), 0.0)
    g = SparseGridFunction.build(hat, 1, 1, 3, 1e-8, ZERO_BOUNDARY)
    assert g.size() == 3
    keys, sur = g.nodes()
    d = {int(k[0]): float(s[0]) for k, s in zip(keys, sur)}
    assert abs(d[1] - 1.0) <= 1e-15 and abs(d[2]) < 1e-15 and abs(d[3]) < 1e-15


def test_monotone_refinement_subset():
    # test_sparse_grid.cpp:179-187
    f = lambda x: np.exp(-10.0 * (x[:, 0] - 0.4) ** 2) * (1.0 + 0.5 * np.sin(4.0 * x[:, 1]))
    loose = SparseGridFunction.build(f, 2, 1, 6, 1e-2, MODIFIED_LINEAR)
    tight = SparseGridFunction.build(f, 2, 1, 6, 1e-4, MODIFIED_LINEAR)
    assert loose.size() <= tight.size()
    kt = {tuple(k) for k in tight.nodes()[0].tolist()}
    assert all(tuple(k) in kt for k in loose.nodes()[0].tolist())


def test_vector_valued_refinement_uses_sup_norm():
    # test_sparse_grid.cpp:189-208
    f = lambda x: np.stack([0.01 * x[:, 0], np.exp(-60.0 * (x[:, 0] - 0.7) ** 2)], axis=1)
    g = lambda x: np.stack([0.01 * x[:, 0], np.zeros(len(x))], axis=1)
    a = SparseGridFunction.build(f, 1, 2, 6, 1e-3, MODIFIED_LINEAR)
    b = SparseGridFunction.build(g, 1, 2, 6, 1e-3, MODIFIED_LINEAR)
    assert a.size() > b.size()


def test_build_reports_offending_point_on_nan():
    # test_sparse_grid.cpp:210-225
    f = lambda x: np.where(x[:, 0] == 0.25, np.nan, x[:, 0])
    with pytest.raises(BuildError) as ei:
        SparseGridFunction.build(f, 1, 1, 3, 0.0, ZERO_BOUNDARY)
    assert len(ei.value.point) == 1 and ei.value.point[0] == 0.25
    assert "0.25" in str(ei.value)


def test_build_validates_options():
    f = wl("wl_constant")
    for args in ((0, 1, 2, 0.0), (1, 0, 2, 0.0), (1, 1, 0, 0.0), (1, 1, 2, -1.0), (1, 1, 31, 0.0)):
        with pytest.raises(InvalidArgument):
            SparseGridFunction.build(f, args[0], args[1], args[2], args[3], ZERO_BOUNDARY)


def test_from_nodes_validation():
    keys = np.array([[1, 1], [2, 1]], dtype=np.uint32)
    sur = np.zeros((2, 1))
    g = SparseGridFunction.from_nodes(2, 1, 3, 0.0, ZERO_BOUNDARY, keys, sur)
    assert g.size() == 2
    with pytest.raises(InvalidArgument):  # duplicate key (sparse_grid.hpp:174-175)
        SparseGridFunction.from_nodes(2, 1, 3, 0.0, ZERO_BOUNDARY, np.array([[1, 1], [1, 1]], dtype=np.uint32),
                                      sur)
    with pytest.raises(InvalidArgument):  # heap key 0 / level > 30
        SparseGridFunction.from_nodes(1, 1, 3, 0.0, ZERO_BOUNDARY, np.array([[0]], dtype=np.uint32), np.zeros((1, 1)))
    with pytest.raises(InvalidArgument):
        SparseGridFunction.from_nodes(1, 1, 3, 0.0, ZERO_BOUNDARY, np.array([[1 << 30]], dtype=np.uint32),
                                      np.zeros((1, 1)))
    with pytest.raises(InvalidArgument):
        SparseGridFunction.from_nodes(2, 1, 3, 0.0, ZERO_BOUNDARY, keys, np.zeros((3, 1)))


def test_append_rejects_duplicates_and_rolls_back():
    keys = np.array([[1]], dtype=np.uint32)
    g = SparseGridFunction.from_nodes(1, 1, 3, 0.0, ZERO_BOUNDARY, keys, np.ones((1, 1)))
    g.append(np.array([[2], [3]], dtype=np.uint32), np.zeros((2, 1)))
    assert g.size() == 3
    with pytest.raises(InvalidArgument):
        g.append(np.array([[4], [2]], dtype=np.uint32), np.zeros((2, 1)))
    assert g.size() == 3


# --------------------------------------------------------------- HDMR

def small_parts():
    keep, ctx = int_ctx(3)
    f = wl("wl_coupled")
    fam = [(), (0,), (1,), (2,), (0, 1)]
    b = W.telescoping_b(fam)
    slots = []
    for u, bu in zip(fam, b):
        g = None
        if u:
            g = SparseGridFunction.build(lambda x, u=u: np.sum(np.exp(-x), axis=1), len(u), 1, 3, 0.0,
                                         MODIFIED_LINEAR)
        slots.append((u, bu, g))
    return slots


def test_hdmr_create_and_info():
    slots = small_parts()
    vec = VectorizedDdsg.compile(3, 1, [1.5], slots)
    info = vec.info()
    assert info["n_slots"] == 5
    assert info["n_active"] == sum(1 for _, b, _ in slots if b != 0)


def test_hdmr_create_validation():
    slots = small_parts()
    with pytest.raises(InvalidArgument):  # empty index must come first
        VectorizedDdsg.compile(3, 1, [1.0], slots[1:])
    with pytest.raises(InvalidArgument):  # not (order, lex) sorted
        VectorizedDdsg.compile(3, 1, [1.0], [slots[0], slots[2], slots[1]] + slots[3:])
    with pytest.raises(InvalidArgument):  # closure: {0,1} without {1} (ddsg_eval.hpp:63-70)
        VectorizedDdsg.compile(3, 1, [1.0], [slots[0], slots[1], slots[3], slots[4]])
    with pytest.raises(InvalidArgument):  # grid dimension != |u|
        VectorizedDdsg.compile(3, 1, [1.0], [slots[0], ((0,), 1, slots[4][2])])
    with pytest.raises(InvalidArgument):  # dimension id out of range
        VectorizedDdsg.compile(2, 1, [1.0], [slots[0], ((2,), 1, slots[1][2])])


@needs_ref
def test_hdmr_quadrature_matches_reference():
    slots = small_parts()
    vec = VectorizedDdsg.compile(3, 1, [1.5], slots)
    grids = [O.ref_from_nodes(len(u), 1, MODIFIED_LINEAR, 3, 0.0, *g.nodes()) if g is not None else None
             for u, b, g in slots]
    ref = O.RefHdmr(3, 1, np.array([1.5]), [(u, b) for u, b, _ in slots], grids)
    assert np.array_equal(bits(vec.quadrature()), bits(ref.quadrature()))


def test_config_shapes():
    assert W.build_grid(W.CONFIGS[1]).size() == 769
    fam = W.hdmr_family(W.CONFIGS[4])
    b = W.telescoping_b(fam)
    assert len(fam) == 146 and b[0] == -54
    assert all(bj == -8 for u, bj in zip(fam, b) if len(u) == 1 and u[0] < 10)
    fam5 = W.hdmr_family(W.CONFIGS[5])
    assert len(fam5) == 601
    b5 = W.telescoping_b(fam5)
    assert sum(1 for v in b5 if v != 0) == 519
