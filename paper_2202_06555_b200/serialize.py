"""JSON documents of the reference's schema (serialize.hpp:19-145), loaded
straight into this package's objects.

Schema version 1, type tags "sparse_grid" / "ddsg"; nodes as
{levels, indices, surplus}.  Floats are written with Python's shortest
round-trip repr and parsed with correctly rounded float(), so surpluses
round-trip bit for bit in both directions (the reference's guarantee,
serialize.hpp:3-5); documents written by the reference load here and ours
load in the reference (tests/test_serialize.py).
"""
from __future__ import annotations

import json
from typing import Any, Dict, List, Optional, Tuple

import numpy as np

from .ddsg import MODIFIED_LINEAR, ZERO_BOUNDARY, InvalidArgument, SparseGridFunction, VectorizedDdsg

SCHEMA_VERSION = 1  # serialize.hpp:19
_MODES = {"zero_boundary": ZERO_BOUNDARY, "modified_linear": MODIFIED_LINEAR}
_MODE_NAMES = {v: k for k, v in _MODES.items()}


def _heap_keys(levels: List[int], indices: List[int]) -> List[int]:
    """heap_key (grid_index.hpp:31-38) with its validation."""
    out = []
    for l, i in zip(levels, indices):
        if l < 1 or l > 30:
            raise InvalidArgument("heap_key: level out of range [1,30]")
        if i % 2 == 0 or i < 1 or i > (1 << l) - 1:
            raise InvalidArgument(f"heap_key: index must be odd in [1, 2^l - 1], got l={l} i={i}")
        out.append((1 << (l - 1)) + (i - 1) // 2)
    return out


def grid_to_json(grid: SparseGridFunction) -> Dict[str, Any]:
    """to_json(SparseGridFunction) (serialize.hpp:31-52), nodes in stored order."""
    keys, sur = grid.nodes()
    lv = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64) + 1
    idx = 2 * (keys.astype(np.int64) - (np.int64(1) << (lv - 1))) + 1
    nodes = [{"levels": lv[i].tolist(), "indices": idx[i].tolist(), "surplus": sur[i].tolist()}
             for i in range(keys.shape[0])]
    return {"schema_version": SCHEMA_VERSION, "type": "sparse_grid", "dim": grid.dim, "out_dim": grid.out_dim,
            "max_level": grid.max_level, "eps_gamma": grid.eps_gamma,
            "boundary_mode": _MODE_NAMES[grid.boundary_mode], "nodes": nodes}


def grid_from_json(doc: Dict[str, Any]) -> SparseGridFunction:
    """sparse_grid_from_json (serialize.hpp:54-77)."""
    if doc.get("schema_version") != SCHEMA_VERSION:
        raise InvalidArgument("sparse grid document: unsupported schema version")
    if doc.get("type") != "sparse_grid":
        raise InvalidArgument("sparse grid document: wrong type tag")
    dim, m = int(doc["dim"]), int(doc["out_dim"])
    if doc["boundary_mode"] not in _MODES:
        raise InvalidArgument("unknown boundary mode: " + str(doc["boundary_mode"]))
    keys, sur = [], []
    for jn in doc["nodes"]:
        if len(jn["levels"]) != len(jn["indices"]):
            raise InvalidArgument("sparse grid document: levels/indices length mismatch")
        keys.append(_heap_keys(jn["levels"], jn["indices"]))
        sur.append([float(v) for v in jn["surplus"]])
    k = np.array(keys, dtype=np.uint32).reshape(-1, dim)
    s = np.array(sur, dtype=np.float64).reshape(-1, m)
    return SparseGridFunction.from_nodes(dim, m, int(doc["max_level"]), float(doc["eps_gamma"]),
                                         _MODES[doc["boundary_mode"]], k, s)


def ddsg_to_json(d: int, m: int, f_anchor, slots, anchor_coords=None, k_max: Optional[int] = None,
                 rejected: Optional[List[Tuple[int, ...]]] = None) -> Dict[str, Any]:
    """to_json(DdsgFunction) (serialize.hpp:85-110) from (dims, b, grid) slots
    in coeff_b order; cut quadratures recomputed from the grids (their
    values in decompose, hdmr.hpp:428)."""
    anchor_coords = [0.5] * d if anchor_coords is None else list(anchor_coords)
    k_max = max((len(u) for u, _, _ in slots), default=0) if k_max is None else k_max
    accepted = [{"dims": list(u), "grid": grid_to_json(g)} for u, b, g in slots if g is not None]
    coeff = [{"dims": list(u), "b": int(b)} for u, b, _ in slots]
    quads = [{"dims": list(u), "q": (list(map(float, f_anchor)) if g is None else g.quadrature().tolist())}
             for u, b, g in slots]
    return {"schema_version": SCHEMA_VERSION, "type": "ddsg", "dim": d, "out_dim": m, "k_max": k_max,
            "anchor": {"coords": anchor_coords, "f_anchor": [float(v) for v in f_anchor]},
            "accepted": accepted, "rejected": [list(z) for z in (rejected or [])], "coeff_b": coeff,
            "cut_quadratures": quads}


def ddsg_from_json(doc: Dict[str, Any]):
    """ddsg_from_json (serialize.hpp:112-145) + compile: returns
    (VectorizedDdsg, slots) with slots = [(dims, b, grid or None)] in
    coeff_b order."""
    if doc.get("schema_version") != SCHEMA_VERSION:
        raise InvalidArgument("ddsg document: unsupported schema version")
    if doc.get("type") != "ddsg":
        raise InvalidArgument("ddsg document: wrong type tag")
    d, m = int(doc["dim"]), int(doc["out_dim"])

    def index(dims):
        u = tuple(sorted(int(v) for v in dims))
        if len(set(u)) != len(u):
            raise InvalidArgument("component index: duplicate dimension")
        if u and (u[0] < 0 or u[-1] >= d):
            raise InvalidArgument("component index: dimension id out of range")
        return u

    grids = {index(e["dims"]): grid_from_json(e["grid"]) for e in doc["accepted"]}
    coeff = sorted(((index(e["dims"]), int(e["b"])) for e in doc["coeff_b"]), key=lambda t: (len(t[0]), t[0]))
    slots = []
    for u, b in coeff:
        if u and u not in grids:
            raise InvalidArgument("vectorized ddsg: coefficient for a non-accepted index")
        slots.append((u, b, grids.get(u)))
    fa = np.array(doc["anchor"]["f_anchor"], dtype=np.float64)
    return VectorizedDdsg.compile(d, m, fa, slots), slots


def dumps(doc: Dict[str, Any]) -> str:
    return json.dumps(doc, allow_nan=False)


def loads(text: str) -> Dict[str, Any]:
    return json.loads(text)
