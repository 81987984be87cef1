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


# ---------------------------------------------------- the C-ABI loader / writer

import json as _json
import re

from paper_2202_06555_b200.ddsg import VectorizedDdsg

_NUM = re.compile(r'-?(?:0|[1-9]\d*)(?:\.\d+)?(?:[eE][+-]?\d+)?')


def _tokens(text: str):
    """Number tokens of a JSON text in document order (both writers sort object
    keys and keep array order, so equal documents give equal sequences)."""
    out, i = [], 0
    in_str = False
    while i < len(text):
        c = text[i]
        if in_str:
            if c == "\\":
                i += 2
                continue
            if c == '"':
                in_str = False
            i += 1
            continue
        if c == '"':
            in_str = True
            i += 1
            continue
        mt = _NUM.match(text, i)
        if mt and (c == "-" or c.isdigit()):
            out.append(mt.group(0))
            i = mt.end()
            continue
        i += 1
    return out


@needs_ref_json
def test_c_abi_grid_document_text_matches_reference_writer():
    """ddsg_grid_to_json writes the same numbers, digit for digit, as the
    reference's nlohmann dump (shortest round-trip, fixed/scientific layout)."""
    f = lambda x: np.exp(x[:, 0]) * np.sin(5.0 * x[:, 1]) + x[:, 1] * 1e-7 - 3.0e5 * x[:, 0] ** 9
    g = SparseGridFunction.build(f, 2, 1, 6, 1e-9, MODIFIED_LINEAR)
    rg = O.ref_from_nodes(2, 1, MODIFIED_LINEAR, 6, 1e-9, *g.nodes())
    ref_text = O.ref().ref_grid_to_json(rg.h).decode()
    ours = g.to_json()
    assert _json.loads(ours) == _json.loads(ref_text)
    t_ref, t_ours = _tokens(ref_text), _tokens(ours)
    assert len(t_ref) == len(t_ours) > 100
    mismatch = [(a, b) for a, b in zip(t_ref, t_ours) if a != b]
    assert not mismatch, mismatch[:5]


@needs_ref_json
def test_c_abi_ddsg_document_round_trip_keeps_every_field():
    """Reference decompose (with a rejected set) -> its document -> our C-ABI
    loader -> our writer: the same document, number for number; the
    evaluator's slots equal the reference's coeff_b family bit for bit."""
    keep, ctx = int_ctx(4)
    fa, parts, text = O.ref_decompose(4, 1, 2, 4, wl("wl_coupled"), ctx, eps_eta=1e-3, eps_gamma=1e-5,
                                      want_json=True)
    ref_doc = _json.loads(text)
    vec = VectorizedDdsg.from_json(text)
    assert [s[0] for s in vec.slots] == [u for u, _, _, _ in parts]
    assert [s[1] for s in vec.slots] == [b for _, b, _, _ in parts]
    for (u, b, g), (_, _, k, s) in zip(vec.slots, parts):
        if g is not None:
            k1, s1 = g.nodes()
            assert np.array_equal(k1, k) and np.array_equal(bits(s1), bits(s))
    k_max, coords, fa2, rej, q = vec.document()
    assert k_max == ref_doc["k_max"] and coords.tolist() == ref_doc["anchor"]["coords"]
    assert np.array_equal(bits(fa2), bits(fa))
    assert [list(u) for u in rej] == ref_doc["rejected"] and len(rej) > 0
    ours = vec.to_json()
    assert _json.loads(ours) == ref_doc
    assert _tokens(ours) == _tokens(text)


def test_c_abi_json_errors():
    bad_docs = [
        "",                                   # empty
        "{",                                  # truncated
        '{"schema_version": 1, "type": "sparse_grid"} x',  # trailing
        '{"schema_version": 1, "type": "sparse_grid"}',    # missing dim
        '{"schema_version": 1, "type": "sparse_grid", "dim": "2", "out_dim": 1, "nodes": []}',  # wrong type
        '{"schema_version": 1, "type": "sparse_grid", "dim": 1, "out_dim": 1, "max_level": 1, "eps_gamma": 0,'
        ' "boundary_mode": "periodic", "nodes": []}',       # unknown mode
        '{"schema_version": 1, "type": "sparse_grid", "dim": 1, "out_dim": 1, "max_level": 1, "eps_gamma": 0,'
        ' "boundary_mode": "zero_boundary", "nodes": [{"levels": [31], "indices": [1], "surplus": [1.0]}]}',
        '{"schema_version": 1, "type": "sparse_grid", "dim": 1, "out_dim": 1, "max_level": 1, "eps_gamma": 0,'
        ' "boundary_mode": "zero_boundary", "nodes": [{"levels": [1], "indices": [1], "surplus": [1.0, 2.0]}]}',
        '{"schema_version": 1, "type": "sparse_grid", "dim": 1, "out_dim": 1, "max_level": 1, "eps_gamma": 0,'
        ' "boundary_mode": "zero_boundary", "nodes": [{"levels": [1], "indices": [1], "surplus": [1.0]},'
        ' {"levels": [1], "indices": [1], "surplus": [2.0]}]}',  # duplicate key
    ]
    for t in bad_docs:
        with pytest.raises(InvalidArgument):
            SparseGridFunction.from_json(t)
    with pytest.raises(InvalidArgument):  # coefficient for a non-accepted index
        VectorizedDdsg.from_json(_json.dumps({
            "schema_version": 1, "type": "ddsg", "dim": 2, "out_dim": 1, "k_max": 1,
            "anchor": {"coords": [0.5, 0.5], "f_anchor": [1.0]}, "accepted": [], "rejected": [],
            "coeff_b": [{"dims": [], "b": 1}, {"dims": [0], "b": 1}], "cut_quadratures": []}))
    with pytest.raises(InvalidArgument):  # no empty slot
        VectorizedDdsg.from_json(_json.dumps({
            "schema_version": 1, "type": "ddsg", "dim": 2, "out_dim": 1, "k_max": 1,
            "anchor": {"coords": [0.5, 0.5], "f_anchor": [1.0]}, "accepted": [], "rejected": [],
            "coeff_b": [], "cut_quadratures": []}))


def test_c_abi_number_layout_and_escapes():
    """nlohmann's number layout (fixed for decimal exponents in (-4, 15],
    '.0' on integral values, e+XX otherwise; -0.0 keeps its sign) and
    round-trip of every bit pattern class through the C-ABI."""
    vals = [0.0, -0.0, 1.0, -2.5, 0.1, 1e-4, 1e-5, 123456789012345.0, 1e15, 1e16, 5e-324, 2.2250738585072014e-308,
            1.7976931348623157e308, 3.141592653589793, -1.0000000000000002, 0.30000000000000004]
    sur = np.array(vals, dtype=np.float64).reshape(-1, 1)
    keys = np.arange(1, len(vals) + 1, dtype=np.uint32).reshape(-1, 1)
    g = SparseGridFunction.from_nodes(1, 1, 5, 0.0, MODIFIED_LINEAR, keys, sur)
    text = g.to_json()
    doc = _json.loads(text)
    got = np.array([n["surplus"][0] for n in doc["nodes"]])
    assert np.array_equal(bits(got), bits(sur.ravel()))
    for v, want in [(1.0, "1.0"), (-0.0, "-0.0"), (1e-4, "0.0001"), (1e-5, "1e-05"), (1e15, "1e+15"),
                    (123456789012345.0, "123456789012345.0"), (0.1, "0.1"), (-2.5, "-2.5")]:
        assert f'"surplus": [\n        {want}\n      ]' in text or f"[{want}]" in text.replace("\n", "").replace(" ", ""), want
    back = SparseGridFunction.from_json(text)
    k2, s2 = back.nodes()
    assert np.array_equal(k2, keys) and np.array_equal(bits(s2), bits(sur))


# ------------------------------------- committed reference-written policies

from pathlib import Path

_GOLD = Path(__file__).resolve().parent / "golden"
_POLICIES = ["policy_vector3_d2_k2_L5", "policy_coupled_d6_k2_L4_pruned"]


@pytest.mark.parametrize("name", _POLICIES)
def test_reference_policy_document_loads_and_rewrites(name):
    """tests/golden/<name>.json was written by the reference (make_golden.py):
    the C-ABI loader keeps every field, and the writer reproduces every
    number token of the reference's text."""
    text = (_GOLD / f"{name}.json").read_text()
    vec = VectorizedDdsg.from_json(text)
    ours = vec.to_json()
    assert _json.loads(ours) == _json.loads(text)
    assert _tokens(ours) == _tokens(text)


@pytest.mark.gpu
@pytest.mark.parametrize("name", _POLICIES)
def test_reference_policy_document_evaluates_bit_exact_on_gpu(name):
    """analyze's policy load (tools/ddsg.cpp:261-268) through the C-ABI, then
    the GPU evaluation, against the reference's evaluation of the same
    document (committed outputs, make_golden.py): bit for bit, from host
    (pageable, pinned-staged) and device buffers."""
    import torch

    text = (_GOLD / f"{name}.json").read_text()
    ref = np.load(_GOLD / f"{name}.npz")
    vec = VectorizedDdsg.from_json(text)
    y = vec.evaluate_batch(ref["x"])
    assert np.array_equal(bits(y), bits(ref["y"]))
    yd = vec.evaluate_batch(torch.from_numpy(ref["x"]).cuda()).cpu().numpy()
    assert np.array_equal(bits(yd), bits(ref["y"]))
