"""Shared test helpers (fixtures loading, canonical node order, builders)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2202_06555_b200 import _native as N
from paper_2202_06555_b200.ddsg import SparseGridFunction, VectorizedDdsg

GOLDEN = Path(__file__).resolve().parent / "golden"

# |delta| <= 1e-14 + 1e-12 |ref| (north star tolerance).
ATOL = 1e-14
RTOL = 1e-12


def within_tol(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    return np.abs(got - want) <= ATOL + RTOL * np.abs(want)


def bits(a: np.ndarray) -> np.ndarray:
    """Raw IEEE-754 bit patterns (bit-exact comparisons, sign of zero included)."""
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def canonical_perm(keys: np.ndarray) -> np.ndarray:
    lv = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64) + 1
    cols = [keys[:, j] for j in reversed(range(keys.shape[1]))] + [lv.sum(axis=1)]
    return np.lexsort(cols)


def golden_files(kind: str):
    out = []
    for p in sorted(GOLDEN.glob("*.npz")):
        if p.name.startswith("policy_"):  # policy documents: tests/test_serialize.py
            continue
        z = np.load(p)
        if str(z["kind"]) == kind:
            out.append(p)
    return out


def load(p):
    return dict(np.load(p))


def hdmr_slots_from_golden(z, canonical: bool):
    """[(dims, b, (mode, keys, surplus) or None)] in coeff_b order."""
    order, dims, b = z["order"], z["dims"], z["b"]
    slots, off = [], 0
    for s in range(len(order)):
        k = int(order[s])
        u = tuple(int(v) for v in dims[off:off + k])
        off += k
        if k == 0:
            slots.append((u, int(b[s]), None))
            continue
        keys, sur = z[f"keys_{s}"], z[f"surplus_{s}"]
        if canonical:
            p = canonical_perm(keys)
            keys, sur = keys[p], sur[p]
        slots.append((u, int(b[s]), (int(z["mode"]), keys, sur)))
    return slots


def make_vectorized(d, m, f_anchor, slots, max_level=8, eps=0.0):
    """Our VectorizedDdsg from (dims, b, (mode, keys, surplus)) slots."""
    ours = []
    for u, b, g in slots:
        if g is None:
            ours.append((u, b, None))
        else:
            ours.append((u, b, SparseGridFunction.from_nodes(len(u), m, max_level, eps, g[0], g[1], g[2])))
    return VectorizedDdsg.compile(d, m, f_anchor, ours)


def int_ctx(v: int):
    keep = C.c_int(v)
    return keep, C.cast(C.pointer(keep), C.c_void_p).value


def wl(name: str) -> int:
    return N.wl_fn(name)
