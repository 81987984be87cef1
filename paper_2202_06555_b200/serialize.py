"""JSON documents of the reference's schema (serialize.hpp:19-145), loaded
straight into this package's objects.

Parsing and writing happen in the C-ABI (ddsg_grid_from_json /
ddsg_grid_to_json / ddsg_hdmr_from_json / ddsg_hdmr_to_json,
csrc/json_doc.cpp), the same loader the C++ shim uses: schema version 1,
type tags "sparse_grid" / "ddsg", nodes as {levels, indices, surplus};
numbers parsed with correctly rounded strtod and written with shortest
round-trip digits, so surpluses round-trip bit for bit in both directions
(serialize.hpp:3-5).  Documents written by the reference load here and ours
load in the reference (tests/test_serialize.py).
"""
from __future__ import annotations

import json
from typing import Any, Dict, List, Optional, Tuple

import numpy as np

from .ddsg import SparseGridFunction, VectorizedDdsg

SCHEMA_VERSION = 1  # serialize.hpp:17


def _text(doc) -> str:
    return doc if isinstance(doc, str) else json.dumps(doc, allow_nan=False)


def grid_to_json(grid: SparseGridFunction) -> Dict[str, Any]:
    """to_json(SparseGridFunction) (serialize.hpp:31-52), nodes in stored
    order -- written by the C-ABI (ddsg_grid_to_json)."""
    return json.loads(grid.to_json())


def grid_from_json(doc) -> SparseGridFunction:
    """sparse_grid_from_json (serialize.hpp:54-77) through the C-ABI
    (ddsg_grid_from_json); doc: a parsed document or its text."""
    return SparseGridFunction.from_json(_text(doc))


def ddsg_to_json(d: int, m: int, f_anchor, slots, anchor_coords=None, k_max: Optional[int] = None,
                 rejected: Optional[List[Tuple[int, ...]]] = None, cut_quadratures=None) -> Dict[str, Any]:
    """to_json(DdsgFunction) (serialize.hpp:85-110) from (dims, b, grid) slots
    in coeff_b order, written by the C-ABI (ddsg_hdmr_to_json).  Cut
    quadratures default to the grids' quadratures (f_anchor for the empty
    index), which are decompose's values (hdmr.hpp:428)."""
    vec = VectorizedDdsg.compile(d, m, f_anchor, slots)
    anchor_coords = [0.5] * d if anchor_coords is None else list(anchor_coords)
    k_max = max((len(u) for u, _, _ in slots), default=0) if k_max is None else k_max
    if cut_quadratures is None:
        cut_quadratures = np.array([np.asarray(f_anchor, dtype=np.float64) if g is None else g.quadrature()
                                    for _, _, g in slots])
    vec.set_document(k_max, anchor_coords, rejected or [], cut_quadratures)
    return json.loads(vec.to_json())


def ddsg_from_json(doc):
    """ddsg_from_json (serialize.hpp:112-145) + compile through the C-ABI
    (ddsg_hdmr_from_json): returns (VectorizedDdsg, slots) with slots =
    [(dims, b, grid or None)] in coeff_b order."""
    vec = VectorizedDdsg.from_json(_text(doc))
    return vec, vec.slots


def dumps(doc: Dict[str, Any]) -> str:
    return json.dumps(doc, allow_nan=False)


def loads(text: str) -> Dict[str, Any]:
    return json.loads(text)
