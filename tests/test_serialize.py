"""JSON documents of the reference's schema (serialize.hpp) — SURVEY.md §8(f)
row 4.  Documents written by the reference load here with bit-identical
surpluses and vice versa (test_sparse_grid.cpp:246-260, test_hdmr.cpp:315-331)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits, int_ctx, wl
from paper_2202_06555_b200 import serialize as S
from paper_2202_06555_b200.ddsg import MODIFIED_LINEAR, InvalidArgument, SparseGridFunction, uniform_points

REF_JSON = O.ref() is not None and O.ref().ref_json_enabled()
needs_ref_json = pytest.mark.skipif(not REF_JSON, reason="oracle/_ref built without serialize.hpp")


def test_round_trip_ours():
    keep, ctx = int_ctx(2)
    g = SparseGridFunction.build(wl("wl_exp_product"), 2, 1, 4, 1e-4, MODIFIED_LINEAR, ctx=ctx)
    g2 = S.grid_from_json(S.loads(S.dumps(S.grid_to_json(g))))
    k1, s1 = g.nodes()
    k2, s2 = g2.nodes()
    assert np.array_equal(k1, k2) and np.array_equal(bits(s1), bits(s2))
    assert (g2.max_level, g2.eps_gamma, g2.boundary_mode) == (g.max_level, g.eps_gamma, g.boundary_mode)


@needs_ref_json
def test_reference_grid_document_loads_bit_exact():
    # test_sparse_grid.cpp:246-260 target: exp(x0) sin(5 x1) + x1, adaptive
    f = lambda x: np.exp(x[:, 0]) * np.sin(5.0 * x[:, 1]) + x[:, 1]
    g = SparseGridFunction.build(f, 2, 1, 4, 1e-4, MODIFIED_LINEAR)
    rg = O.ref_from_nodes(2, 1, MODIFIED_LINEAR, 4, 1e-4, *g.nodes())
    text = O.ref().ref_grid_to_json(rg.h).decode()
    ours = S.grid_from_json(S.loads(text))
    k1, s1 = ours.nodes()
    k2, s2 = rg.nodes(2, 1)
    assert np.array_equal(k1, k2) and np.array_equal(bits(s1), bits(s2))
    # and our document loads in the reference, bit for bit
    h = C.c_void_p()
    assert O.ref().ref_grid_from_json(S.dumps(S.grid_to_json(ours)).encode(), C.byref(h)) == 0
    back = O.RefGrid(h.value)
    k3, s3 = back.nodes(2, 1)
    assert np.array_equal(k3, k1) and np.array_equal(bits(s3), bits(s1))


@needs_ref_json
def test_reference_ddsg_document_round_trip():
    # test_hdmr.cpp:315-331: decompose exp(x0 x1) + x1, k_max 2, L 4, eps_gamma 1e-5
    keep, ctx = int_ctx(4)
    fa, parts, text = O.ref_decompose(4, 1, 2, 4, wl("wl_coupled"), ctx, eps_gamma=1e-5, want_json=True)
    vec, slots = S.ddsg_from_json(S.loads(text))
    assert [u for u, _, _ in slots] == [u for u, _, _, _ in parts]
    assert [b for _, b, _ in slots] == [b for _, b, _, _ in parts]
    for (u, b, g), (_, _, k, s) in zip(slots, parts):
        if g is not None:
            k1, s1 = g.nodes()
            assert np.array_equal(k1, k) and np.array_equal(bits(s1), bits(s))
    # our document -> reference evaluation equals the reference's evaluation of its own document
    mine = S.dumps(S.ddsg_to_json(4, 1, fa, slots))
    h1, h2 = C.c_void_p(), C.c_void_p()
    assert O.ref().ref_hdmr_from_json(text.encode(), C.byref(h1)) == 0
    assert O.ref().ref_hdmr_from_json(mine.encode(), C.byref(h2)) == 0
    x = uniform_points(40, 50, 4)
    y1 = np.empty((50, 1))
    y2 = np.empty((50, 1))
    O.ref().ref_hdmr_eval(h1, x.ctypes.data, 50, y1.ctypes.data, 1)
    O.ref().ref_hdmr_eval(h2, x.ctypes.data, 50, y2.ctypes.data, 1)
    assert np.array_equal(bits(y1), bits(y2))
    O.ref().ref_hdmr_free(h1)
    O.ref().ref_hdmr_free(h2)


def test_schema_validation():
    with pytest.raises(InvalidArgument):
        S.grid_from_json({"schema_version": 2, "type": "sparse_grid"})
    with pytest.raises(InvalidArgument):
        S.grid_from_json({"schema_version": 1, "type": "ddsg"})
    doc = {"schema_version": 1, "type": "sparse_grid", "dim": 1, "out_dim": 1, "max_level": 2, "eps_gamma": 0.0,
           "boundary_mode": "zero_boundary", "nodes": [{"levels": [2], "indices": [2], "surplus": [1.0]}]}
    with pytest.raises(InvalidArgument):  # even index (grid_index.hpp:34-36)
        S.grid_from_json(doc)
