"""ctypes bindings of the CPU oracles (test infrastructure).

  port()  -> oracle/liboracle.so           the C restatement (oracle/ddsg_oracle.c)
  ref()   -> oracle/_ref/libddsg_ref.so    the unmodified reference headers
                                           compiled in place (None if absent)
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
PORT_PATH = ROOT / "oracle" / "liboracle.so"
REF_PATH = ROOT / "oracle" / "_ref" / "libddsg_ref.so"

_p, _i, _i64, _d, _u64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64


def _ptr(a):
    return None if a is None else a.ctypes.data


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not PORT_PATH.exists():
            raise RuntimeError(f"{PORT_PATH} missing: run `make -C oracle port`")
        L = C.CDLL(str(PORT_PATH))
        L.oracle_basis_value.restype = _d
        L.oracle_basis_value.argtypes = [_i, _i, C.c_uint32, _d]
        L.oracle_grid_eval.restype = _i
        L.oracle_grid_eval.argtypes = [_i, _i, _i, _i64, _p, _p, _p, _i64, _p, C.POINTER(_i64)]
        L.oracle_grid_support.restype = _i
        L.oracle_grid_support.argtypes = [_i, _i, _i64, _p, _p, _i64, _p, _p]
        L.oracle_hdmr_eval.restype = _i
        L.oracle_hdmr_eval.argtypes = [_i, _i, _p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _p, C.POINTER(_i64)]
        L.oracle_hdmr_support.restype = _i
        L.oracle_hdmr_support.argtypes = [_i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _p, _p]
        L.oracle_b_coefficients.restype = _i
        L.oracle_b_coefficients.argtypes = [_i, _p, _p, _p]
        L.oracle_uniform_points.restype = None
        L.oracle_uniform_points.argtypes = [_u64, _i64, _i, _p]
        _port = L
    return _port


def ref():
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            return None
        L = C.CDLL(str(REF_PATH))
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_task.restype = _i64
        L.ref_basis_1d.restype = _i
        L.ref_basis_1d.argtypes = [_i, C.c_uint32, _d, _i, C.POINTER(_d)]
        L.ref_heap_key.restype = _i
        L.ref_heap_key.argtypes = [_i, C.c_uint32, C.POINTER(C.c_uint32)]
        L.ref_grid_from_nodes.restype = _i
        L.ref_grid_from_nodes.argtypes = [_i, _i, _i, _i, _d, _i64, _p, _p, C.POINTER(_p)]
        L.ref_grid_build.restype = _i
        L.ref_grid_build.argtypes = [_i, _i, _i, _i, _d, _i, C.c_uint, _p, _p, C.POINTER(_p)]
        L.ref_grid_free.argtypes = [_p]
        L.ref_grid_size.restype = _i64
        L.ref_grid_size.argtypes = [_p]
        L.ref_grid_nodes.argtypes = [_p, _p, _p]
        L.ref_grid_quadrature.restype = _i
        L.ref_grid_quadrature.argtypes = [_p, _p]
        L.ref_grid_eval.restype = _i
        L.ref_grid_eval.argtypes = [_p, _p, _i64, _p, C.c_uint]
        L.ref_hdmr_from_parts.restype = _i
        L.ref_hdmr_from_parts.argtypes = [_i, _i, _p, _i, _p, _p, _p, _p, C.POINTER(_p)]
        L.ref_hdmr_free.argtypes = [_p]
        for nm in ("ref_hdmr_eval", "ref_hdmr_eval_flat"):
            getattr(L, nm).restype = _i
            getattr(L, nm).argtypes = [_p, _p, _i64, _p, C.c_uint]
        L.ref_hdmr_eval_one.restype = _i
        L.ref_hdmr_eval_one.argtypes = [_p, _p, _p, C.POINTER(_u64)]
        L.ref_hdmr_eval_naive.restype = _i
        L.ref_hdmr_eval_naive.argtypes = [_p, _p, _i64, _p]
        L.ref_hdmr_quadrature.restype = _i
        L.ref_hdmr_quadrature.argtypes = [_p, _p]
        L.ref_decompose.restype = _i
        L.ref_decompose.argtypes = [_i, _i, _i, _d, _d, _i, _d, _i, C.c_uint, _p, _p, C.POINTER(_p)]
        L.ref_decomp_free.argtypes = [_p]
        L.ref_decomp_n_slots.restype = _i
        L.ref_decomp_n_slots.argtypes = [_p]
        L.ref_decomp_slot.restype = _p
        L.ref_decomp_slot.argtypes = [_p, _i, C.POINTER(C.c_int32), _p, C.POINTER(C.c_int32)]
        L.ref_decomp_anchor.argtypes = [_p, _p]
        L.ref_uniform_points.argtypes = [_i, _i64, _u64, _p]
        L.ref_sg_node_count_bruteforce.restype = _u64
        L.ref_sg_node_count_bruteforce.argtypes = [_i, _i]
        L.ref_default_workers.restype = C.c_uint
        L.ref_irbc_refresh.restype = _i
        L.ref_irbc_refresh.argtypes = [_i, _i, _p, _p, _p, _p, C.POINTER(_d)]
        L.ref_irbc_steady_lambda.restype = _i
        L.ref_irbc_steady_lambda.argtypes = [_i, _i, _p, _p, C.POINTER(_d)]
        L.ref_irbc_foc_residuals.restype = _i
        L.ref_irbc_foc_residuals.argtypes = [_p, _p, _i, _i, _p, _p, _i64, _p, _p, _p, C.c_uint, _p, _p]
        L.ref_irbc_foc_jacobian.restype = _i
        L.ref_irbc_foc_jacobian.argtypes = [_p, _p, _i, _i, _p, _p, _i64, _p, _p, _p, _p, _d, _p]
        L.ref_irbc_euler_errors.restype = _i
        L.ref_irbc_euler_errors.argtypes = [_p, _p, _i, _i, _p, _p, _i64, _p, C.c_uint, _p, _p, C.POINTER(_u64)]
        L.ref_json_enabled.restype = _i
        if L.ref_json_enabled():
            L.ref_grid_to_json.restype = C.c_char_p
            L.ref_grid_to_json.argtypes = [_p]
            L.ref_grid_from_json.restype = _i
            L.ref_grid_from_json.argtypes = [C.c_char_p, C.POINTER(_p)]
            L.ref_decomp_to_json.restype = C.c_char_p
            L.ref_decomp_to_json.argtypes = [_p]
            L.ref_hdmr_from_json.restype = _i
            L.ref_hdmr_from_json.argtypes = [C.c_char_p, C.POINTER(_p)]
        _ref = L
    return _ref


# ------------------------------------------------------------ port helpers

def port_grid_eval(dim, m, mode, keys, surplus, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    y = np.empty((n, m), dtype=np.float64)
    bad = _i64(-1)
    rc = port().oracle_grid_eval(dim, m, mode, keys.shape[0], _ptr(np.ascontiguousarray(keys, dtype=np.uint32)),
                                 _ptr(np.ascontiguousarray(surplus, dtype=np.float64)), _ptr(x), n, _ptr(y),
                                 C.byref(bad))
    return rc, y, bad.value


def port_grid_support(dim, mode, keys, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    nnz = np.empty(n, dtype=np.int64)
    h = np.empty(n, dtype=np.uint64)
    rc = port().oracle_grid_support(dim, mode, keys.shape[0], _ptr(np.ascontiguousarray(keys, dtype=np.uint32)),
                                    _ptr(x), n, _ptr(nnz), _ptr(h))
    assert rc == 0
    return nnz, h


def _flatten_slots(slots, m):
    """slots: list of (dims, b, (mode, keys, surplus) or None)."""
    order = np.array([len(s[0]) for s in slots], dtype=np.int32)
    dims = np.array([v for s in slots for v in s[0]] or [0], dtype=np.int32)
    b = np.array([s[1] for s in slots], dtype=np.int32)
    gmode = np.array([(s[2][0] if s[2] is not None else 0) for s in slots], dtype=np.int32)
    gn = np.array([(s[2][1].shape[0] if s[2] is not None else 0) for s in slots], dtype=np.int64)
    keys = [np.ascontiguousarray(s[2][1], dtype=np.uint32).ravel() for s in slots if s[2] is not None]
    sur = [np.ascontiguousarray(s[2][2], dtype=np.float64).ravel() for s in slots if s[2] is not None]
    keys = np.concatenate(keys) if keys else np.zeros(1, dtype=np.uint32)
    sur = np.concatenate(sur) if sur else np.zeros(1, dtype=np.float64)
    return order, dims, b, gmode, gn, keys, sur


def port_hdmr_eval(d, m, f_anchor, slots, x):
    order, dims, b, gmode, gn, keys, sur = _flatten_slots(slots, m)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    y = np.empty((n, m), dtype=np.float64)
    bad = _i64(-1)
    fa = np.ascontiguousarray(f_anchor, dtype=np.float64)
    rc = port().oracle_hdmr_eval(d, m, _ptr(fa), len(slots), _ptr(order), _ptr(dims), _ptr(b), _ptr(gmode), _ptr(gn),
                                 _ptr(keys), _ptr(sur), _ptr(x), n, _ptr(y), C.byref(bad))
    return rc, y, bad.value


def port_hdmr_support(d, m, slots, x):
    order, dims, b, gmode, gn, keys, sur = _flatten_slots(slots, m)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    nnz = np.empty(n, dtype=np.int64)
    h = np.empty(n, dtype=np.uint64)
    rc = port().oracle_hdmr_support(d, m, len(slots), _ptr(order), _ptr(dims), _ptr(b), _ptr(gmode), _ptr(gn),
                                    _ptr(keys), _ptr(sur), _ptr(x), n, _ptr(nnz), _ptr(h))
    assert rc == 0
    return nnz, h


def port_uniform_points(seed, n, dim):
    out = np.empty((n, dim), dtype=np.float64)
    port().oracle_uniform_points(seed, n, dim, _ptr(out))
    return out


# ------------------------------------------------------------- ref helpers

class RefGrid:
    def __init__(self, h):
        self.h = C.c_void_p(h)

    def __del__(self):
        if self.h.value:
            ref().ref_grid_free(self.h)

    def size(self):
        return ref().ref_grid_size(self.h)

    def nodes(self, dim, m):
        n = self.size()
        keys = np.empty((n, dim), dtype=np.uint32)
        sur = np.empty((n, m), dtype=np.float64)
        ref().ref_grid_nodes(self.h, _ptr(keys), _ptr(sur))
        return keys, sur

    def eval(self, x, m, workers=1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty((x.shape[0], m), dtype=np.float64)
        rc = ref().ref_grid_eval(self.h, _ptr(x), x.shape[0], _ptr(y), workers)
        return rc, y

    def quadrature(self, m):
        q = np.empty(m, dtype=np.float64)
        assert ref().ref_grid_quadrature(self.h, _ptr(q)) == 0
        return q


def ref_from_nodes(dim, m, mode, max_level, eps, keys, surplus):
    h = _p()
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    surplus = np.ascontiguousarray(surplus, dtype=np.float64)
    rc = ref().ref_grid_from_nodes(dim, m, mode, max_level, eps, keys.shape[0], _ptr(keys), _ptr(surplus), C.byref(h))
    assert rc == 0, ref().ref_last_error()
    return RefGrid(h.value)


def ref_build(dim, m, mode, max_level, eps, fn_addr, ctx=None, norm=0, workers=1):
    h = _p()
    rc = ref().ref_grid_build(dim, m, mode, max_level, eps, norm, workers, C.c_void_p(fn_addr), ctx, C.byref(h))
    if rc != 0:
        return rc, ref().ref_last_error().decode()
    return 0, RefGrid(h.value)


class RefHdmr:
    def __init__(self, d, m, f_anchor, slots, grids):
        """slots: list of (dims, b); grids: list of RefGrid or None."""
        order = np.array([len(s[0]) for s in slots], dtype=np.int32)
        dims = np.array([v for s in slots for v in s[0]] or [0], dtype=np.int32)
        b = np.array([s[1] for s in slots], dtype=np.int32)
        gp = (C.c_void_p * len(slots))(*[(g.h.value if g is not None else None) for g in grids])
        self._keep = grids
        fa = np.ascontiguousarray(f_anchor, dtype=np.float64)
        h = _p()
        rc = ref().ref_hdmr_from_parts(d, m, _ptr(fa), len(slots), _ptr(order), _ptr(dims), _ptr(b),
                                       C.cast(gp, C.c_void_p), C.byref(h))
        assert rc == 0, ref().ref_last_error()
        self.h = h
        self.d, self.m = d, m

    def __del__(self):
        if self.h.value:
            ref().ref_hdmr_free(self.h)

    def eval(self, x, workers=1, flat=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty((x.shape[0], self.m), dtype=np.float64)
        fn = ref().ref_hdmr_eval_flat if flat else ref().ref_hdmr_eval
        rc = fn(self.h, _ptr(x), x.shape[0], _ptr(y), workers)
        return rc, y

    def eval_naive(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty((x.shape[0], self.m), dtype=np.float64)
        rc = ref().ref_hdmr_eval_naive(self.h, _ptr(x), x.shape[0], _ptr(y))
        return rc, y

    def eval_calls(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.m, dtype=np.float64)
        calls = _u64(0)
        rc = ref().ref_hdmr_eval_one(self.h, _ptr(x), _ptr(y), C.byref(calls))
        return rc, y, calls.value

    def quadrature(self):
        q = np.empty(self.m, dtype=np.float64)
        assert ref().ref_hdmr_quadrature(self.h, _ptr(q)) == 0
        return q


def ref_decompose(d, m, k_max, max_level, fn_addr, ctx=None, eps_rho=0.0, eps_eta=0.0, eps_gamma=0.0, mode=1,
                  want_json=False):
    """Runs the reference decompose (center anchor) and returns
    (f_anchor, [(dims, b, keys, surplus) ...] in coeff_b order)."""
    L = ref()
    h = _p()
    rc = L.ref_decompose(d, m, k_max, eps_rho, eps_eta, max_level, eps_gamma, mode, 1, C.c_void_p(fn_addr), ctx,
                         C.byref(h))
    assert rc == 0, L.ref_last_error()
    fa = np.empty(m, dtype=np.float64)
    L.ref_decomp_anchor(h, _ptr(fa))
    out = []
    dims_buf = np.zeros(64, dtype=np.int32)
    for s in range(L.ref_decomp_n_slots(h)):
        order, b = C.c_int32(), C.c_int32()
        g = L.ref_decomp_slot(h, s, C.byref(order), _ptr(dims_buf), C.byref(b))
        dims = tuple(int(v) for v in dims_buf[: order.value])
        if g:
            rg = RefGrid(g)
            keys, sur = rg.nodes(order.value, m)
            out.append((dims, b.value, keys, sur))
        else:
            out.append((dims, b.value, None, None))
    text = L.ref_decomp_to_json(h).decode() if want_json else None
    L.ref_decomp_free(h)
    return (fa, out, text) if want_json else (fa, out)


# ------------------------------------------------------------- IRBC callers

def _irbc_scal(p):
    return np.array([p.beta, p.alpha, p.delta, p.sigma, p.rho_a, p.phi_adj, p.gamma_base, p.lna_half_width,
                     p.k_lo, p.k_hi], dtype=np.float64)


def _irbc_gamma(p):
    return np.ascontiguousarray(p.gamma, dtype=np.float64) if p.gamma else None


def ref_irbc_refresh(p):
    """(gamma, tau, A) from the reference's refresh_derived (irbc.hpp:59-92)."""
    n = p.countries
    g, t, A = np.empty(n), np.empty(n), _d()
    sc, gi = _irbc_scal(p), _irbc_gamma(p)
    rc = ref().ref_irbc_refresh(n, p.variant, _ptr(sc), _ptr(gi), _ptr(g), _ptr(t), C.byref(A))
    return rc, g, t, A.value


def ref_irbc_steady_lambda(p):
    out = _d()
    sc, gi = _irbc_scal(p), _irbc_gamma(p)
    rc = ref().ref_irbc_steady_lambda(p.countries, p.variant, _ptr(sc), _ptr(gi), C.byref(out))
    assert rc == 0, ref().ref_last_error()
    return out.value


def _policy_handles(policy):
    if isinstance(policy, RefHdmr):
        return policy.h, None
    return None, policy.h


def ref_irbc_foc_residuals(policy, p, a, k, cand, workers=1):
    a, k, cand = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, k, cand))
    n, pd = cand.shape
    res = np.empty((n, pd))
    cl = np.empty(n, dtype=np.int32)
    h, g = _policy_handles(policy)
    sc, gi = _irbc_scal(p), _irbc_gamma(p)
    rc = ref().ref_irbc_foc_residuals(h, g, p.countries, p.variant, _ptr(sc), _ptr(gi), n,
                                      _ptr(a), _ptr(k), _ptr(cand), workers, _ptr(res), _ptr(cl))
    assert rc == 0, ref().ref_last_error()
    return res, cl


def ref_irbc_foc_jacobian(policy, p, a, k, z, r0, fd_epsilon=1e-7):
    a, k, z, r0 = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, k, z, r0))
    n, pd = z.shape
    jac = np.empty((n, pd, pd))
    h, g = _policy_handles(policy)
    sc, gi = _irbc_scal(p), _irbc_gamma(p)
    rc = ref().ref_irbc_foc_jacobian(h, g, p.countries, p.variant, _ptr(sc), _ptr(gi), n,
                                     _ptr(a), _ptr(k), _ptr(z), _ptr(r0), fd_epsilon, _ptr(jac))
    assert rc == 0, ref().ref_last_error()
    return jac


def ref_irbc_euler_errors(policy, p, xs, workers=1):
    """(errs, mean, worst, clamp_count) — solver.hpp:377-436 on samples xs."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    n = xs.shape[0]
    errs, stats, cl = np.empty(n), np.empty(2), _u64()
    h, g = _policy_handles(policy)
    sc, gi = _irbc_scal(p), _irbc_gamma(p)
    rc = ref().ref_irbc_euler_errors(h, g, p.countries, p.variant, _ptr(sc), _ptr(gi), n,
                                     _ptr(xs), workers, _ptr(errs), _ptr(stats), C.byref(cl))
    assert rc == 0, ref().ref_last_error()
    return errs, stats[0], stats[1], cl.value
