"""Generates the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists and `make -C oracle ref` has built
oracle/_ref/libddsg_ref.so):   python tests/golden/make_golden.py

Every fixture is produced by the unmodified reference code
(SparseGridFunction::build / interpolate, decompose, VectorizedDdsg::
evaluate_batch, evaluate_naive), with the reference's own seeded point
generator (proj/tests/oracles.hpp:45-53).  Grids are stored in the
reference's stored order AND re-evaluated by the reference after canonical
reordering, so the fixtures pin both the oracle (stored order) and the GPU
path (canonical order).  Targets are the C functions of
libddsg_workloads.so (same bits for both builders).
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

import oracle_lib as O  # noqa: E402
from paper_2202_06555_b200 import _native as N  # noqa: E402


def canonical_perm(keys: np.ndarray) -> np.ndarray:
    """Stored -> canonical order: (level sum, heap-key lexicographic)."""
    lv = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64) + 1
    cols = [keys[:, j] for j in reversed(range(keys.shape[1]))] + [lv.sum(axis=1)]
    return np.lexsort(cols)


def edge_points(dim: int, n_random: int, seed: int) -> np.ndarray:
    """Seeded points plus the domain edges: 0, 1 and dyadic cell boundaries."""
    pts = np.empty((n_random, dim))
    O.ref().ref_uniform_points(dim, n_random, seed, pts.ctypes.data)
    rng = np.random.default_rng(seed)
    special = np.array([0.0, 1.0, 0.5, 0.25, 0.75, 0.125, 1.0 / 3.0, 1.0 - 2.0**-53, 2.0**-40])
    e = rng.choice(special, size=(16, dim))
    return np.concatenate([pts, e, np.zeros((1, dim)), np.ones((1, dim))])


def grid_case(name, fn, dim, m, L, eps, mode, ctx_dim=None, n=48, seed=0):
    ctx = None
    keep = None
    if ctx_dim is not None:
        keep = C.c_int(ctx_dim)
        ctx = C.cast(C.pointer(keep), C.c_void_p)
    rc, g = O.ref_build(dim, m, mode, L, eps, N.wl_fn(fn), ctx)
    assert rc == 0, g
    keys, sur = g.nodes(dim, m)
    x = edge_points(dim, n, seed)
    rc, y_stored = g.eval(x, m)
    assert rc == 0
    perm = canonical_perm(keys)
    gc = O.ref_from_nodes(dim, m, mode, L, eps, keys[perm], sur[perm])
    rc, y_canon = gc.eval(x, m)
    assert rc == 0
    np.savez_compressed(HERE / f"{name}.npz", kind="grid", dim=dim, m=m, mode=mode, max_level=L, eps=eps,
                        keys=keys, surplus=sur, x=x, y_stored=y_stored, y_canonical=y_canon,
                        quadrature=g.quadrature(m))
    print(name, keys.shape[0], "nodes")


def hdmr_case(name, fn, d, m, k_max, L, eps_gamma=0.0, eps_eta=0.0, ctx_dim=None, n=48, seed=0):
    ctx = None
    keep = None
    if ctx_dim is not None:
        keep = C.c_int(ctx_dim)
        ctx = C.cast(C.pointer(keep), C.c_void_p)
    fa, slots = O.ref_decompose(d, m, k_max, L, N.wl_fn(fn), ctx, eps_eta=eps_eta, eps_gamma=eps_gamma)
    x = edge_points(d, n, seed)
    grids, grids_c = [], []
    arrays = {}
    for s, (dims, b, keys, sur) in enumerate(slots):
        if keys is None:
            grids.append(None)
            grids_c.append(None)
            continue
        grids.append(O.ref_from_nodes(len(dims), m, 1, L, eps_gamma, keys, sur))
        perm = canonical_perm(keys)
        grids_c.append(O.ref_from_nodes(len(dims), m, 1, L, eps_gamma, keys[perm], sur[perm]))
        arrays[f"keys_{s}"] = keys
        arrays[f"surplus_{s}"] = sur
    h = O.RefHdmr(d, m, fa, [(s[0], s[1]) for s in slots], grids)
    hc = O.RefHdmr(d, m, fa, [(s[0], s[1]) for s in slots], grids_c)
    rc, y_stored = h.eval(x, flat=False)
    assert rc == 0
    rc, y_canon = hc.eval(x, flat=False)
    assert rc == 0
    rc, y_naive = h.eval_naive(x)
    assert rc == 0
    order = np.array([len(s[0]) for s in slots], dtype=np.int32)
    dims = np.array([v for s in slots for v in s[0]], dtype=np.int32)
    b = np.array([s[1] for s in slots], dtype=np.int32)
    np.savez_compressed(HERE / f"{name}.npz", kind="hdmr", d=d, m=m, mode=1, max_level=L, eps=eps_gamma,
                        f_anchor=fa, order=order, dims=dims, b=b, x=x, y_stored=y_stored, y_canonical=y_canon,
                        y_naive=y_naive, quadrature=h.quadrature(), **arrays)
    print(name, len(slots), "slots")


def policy_case(name, fn, d, m, k_max, L, eps_gamma=0.0, eps_eta=0.0, ctx_dim=None, n=256, seed=0):
    """A policy document written by the reference (to_json + dump, as
    save_json, serialize.hpp:84-110,147-152) and the reference's evaluation of
    that document after its own ddsg_from_json + compile."""
    ctx = None
    keep = None
    if ctx_dim is not None:
        keep = C.c_int(ctx_dim)
        ctx = C.cast(C.pointer(keep), C.c_void_p)
    _, _, text = O.ref_decompose(d, m, k_max, L, N.wl_fn(fn), ctx, eps_eta=eps_eta, eps_gamma=eps_gamma,
                                 want_json=True)
    (HERE / f"{name}.json").write_text(text)
    h = C.c_void_p()
    assert O.ref().ref_hdmr_from_json(text.encode(), C.byref(h)) == 0
    x = edge_points(d, n, seed)
    y = np.empty((x.shape[0], m))
    assert O.ref().ref_hdmr_eval(h, x.ctypes.data, x.shape[0], y.ctypes.data, 1) == 0
    O.ref().ref_hdmr_free(h)
    np.savez_compressed(HERE / f"{name}.npz", x=x, y=y)
    print(name, len(text), "bytes")


def main():
    if O.ref() is None:
        raise SystemExit("oracle/_ref/libddsg_ref.so missing: make -C oracle ref")
    grid_case("sg_config1_d4_L5", "wl_config1", 4, 1, 5, 0.0, 0, n=64, seed=1001)
    grid_case("sg_roundtrip_d2_L5_zero", "wl_exp_product", 2, 1, 5, 0.0, 0, ctx_dim=2, seed=11)
    grid_case("sg_roundtrip_d2_L5_mod", "wl_exp_product", 2, 1, 5, 0.0, 1, ctx_dim=2, seed=12)
    grid_case("sg_adaptive_bump_d2_L6", "wl_bump", 2, 1, 6, 1e-3, 1, seed=13)
    grid_case("sg_adaptive_coupled_d5_L5", "wl_coupled", 5, 1, 5, 1e-3, 1, ctx_dim=5, seed=14)
    grid_case("sg_vector3_d2_L4", "wl_vector3", 2, 3, 4, 0.0, 1, seed=15)
    hdmr_case("hdmr_coupled_d8_k2_L3", "wl_coupled", 8, 1, 2, 3, ctx_dim=8, seed=321)
    hdmr_case("hdmr_coupled_d4_k2_L4_adaptive", "wl_coupled", 4, 1, 2, 4, eps_gamma=1e-5, ctx_dim=4, seed=8443)
    hdmr_case("hdmr_pruned_d3_k2_L3", "wl_pruned3", 3, 1, 2, 3, eps_eta=1e-4, seed=77)
    hdmr_case("hdmr_vector3_d2_k2_L4", "wl_vector3", 2, 3, 2, 4, seed=61)
    policy_case("policy_vector3_d2_k2_L5", "wl_vector3", 2, 3, 2, 5, eps_gamma=1e-6, seed=62)
    policy_case("policy_coupled_d6_k2_L4_pruned", "wl_coupled", 6, 1, 2, 4, eps_gamma=1e-5, eps_eta=1e-3,
                ctx_dim=6, seed=63)


if __name__ == "__main__":
    main()
