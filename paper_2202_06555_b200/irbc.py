"""Batched IRBC policy callers on the device.

Mirror of the reference's irbc / solver interface (irbc.hpp, solver.hpp):
``IrbcParameters`` / ``make_parameters`` / ``refresh_derived`` /
``steady_state_lambda`` / ``make_shock_quadrature`` keep their names and
meaning, and the three policy consumers take a whole batch of states at
once:

* ``foc_residuals(policy, p, a, k, candidate)`` -> (residuals, clamped):
  irbc.hpp:306-361 for n states, all n * 2(N+1) successor states evaluated
  by one batched policy call;
* ``foc_jacobian(policy, p, a, k, z, r0, fd_epsilon)`` -> jac[n][pdim][pdim]:
  solver.hpp:129-165, (1 + N) * 2(N+1) successor evaluations per state in
  one call (a mu / lambda column leaves the successor states unchanged);
* ``euler_errors(policy, p, n_samples, seed)`` -> EulerErrors:
  solver.hpp:377-436 with the reference's sample stream.

``policy`` is a device interpolant on the canonical state cube: a
``VectorizedDdsg`` (the reference's compiled_evaluator,
time_iteration.hpp:86-91) or a ``SparseGridFunction``; input dim 2N, output
dim pdim.  State / candidate buffers may be numpy arrays or CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .ddsg import InvalidArgument, SparseGridFunction, VectorizedDdsg, _check, _DeviceScope, _ptr, uniform_points

SMOOTH, NONSMOOTH = 0, 1  # irbc.hpp:25 Variant


@dataclass
class IrbcParameters:
    """irbc.hpp:27-53 (same defaults)."""

    countries: int = 2
    beta: float = 0.99
    alpha: float = 0.36
    delta: float = 0.01
    sigma: float = 0.01
    rho_a: float = 0.95
    phi_adj: float = 0.50
    gamma_base: float = 0.25
    gamma: List[float] = field(default_factory=list)
    variant: int = SMOOTH
    lna_half_width: float = 0.4
    k_lo: float = 0.5
    k_hi: float = 1.5
    A: float = 0.0
    tau: List[float] = field(default_factory=list)

    def state_dim(self) -> int:
        return 2 * self.countries

    def policy_dim(self) -> int:
        return self.countries + 1 if self.variant == SMOOTH else 2 * self.countries + 1

    def _c(self):
        """(ctypes struct, gamma buffer, tau buffer) — buffers must outlive the struct."""
        n = max(self.countries, 1)
        g = np.zeros(n, dtype=np.float64)
        t = np.zeros(n, dtype=np.float64)
        if self.gamma:
            g[: len(self.gamma)] = self.gamma[:n]
        if self.tau:
            t[: len(self.tau)] = self.tau[:n]
        s = N.IrbcParamsC(self.countries, self.variant, self.beta, self.alpha, self.delta, self.sigma, self.rho_a,
                          self.phi_adj, self.gamma_base, self.lna_half_width, self.k_lo, self.k_hi, self.A,
                          g.ctypes.data_as(C.POINTER(C.c_double)), t.ctypes.data_as(C.POINTER(C.c_double)))
        return s, g, t


def refresh_derived(p: IrbcParameters) -> None:
    """irbc.hpp:59-92: fills gamma (when empty), A and tau; validates."""
    if p.gamma and len(p.gamma) != p.countries:
        raise InvalidArgument("irbc: gamma length must equal countries")
    s, g, t = p._c()
    _check(N.lib.ddsg_irbc_refresh_derived(C.byref(s), 0 if p.gamma else 1))
    p.gamma = g[: p.countries].tolist()
    p.tau = t[: p.countries].tolist()
    p.A = s.A


def make_parameters(countries: int, variant: int = SMOOTH, gamma_base: float = 0.25) -> IrbcParameters:
    """irbc.hpp:94-101."""
    p = IrbcParameters(countries=countries, variant=variant, gamma_base=gamma_base)
    refresh_derived(p)
    return p


def make_identical_gamma_parameters(countries: int, variant: int, gamma: float) -> IrbcParameters:
    """irbc.hpp:103-112."""
    p = IrbcParameters(countries=countries, variant=variant, gamma_base=gamma, gamma=[gamma] * countries)
    refresh_derived(p)
    return p


def steady_state_lambda(p: IrbcParameters) -> float:
    """irbc.hpp:248-263."""
    s, g, t = p._c()
    out = C.c_double()
    _check(N.lib.ddsg_irbc_steady_state_lambda(C.byref(s), C.byref(out)))
    return out.value


def make_shock_quadrature(countries: int) -> Tuple[np.ndarray, np.ndarray]:
    """irbc.hpp:151-166: 2(N+1) antipodal nodes at +-sqrt(N+1), equal weights
    (node layout [e_1..e_N, e_global]); the kernels generate them implicitly."""
    if countries < 1:
        raise InvalidArgument("shock quadrature: countries must be >= 1")
    n = countries + 1
    r = math.sqrt(float(n))
    nodes = np.zeros((2 * n, n))
    for i in range(n):
        nodes[2 * i, i] = r
        nodes[2 * i + 1, i] = -r
    return nodes, np.full(2 * n, 1.0 / float(2 * n))


def from_canonical(x: np.ndarray, p: IrbcParameters) -> Tuple[np.ndarray, np.ndarray]:
    """irbc.hpp:216-226 (host helper): canonical x[n][2N] -> (a, k)."""
    x = np.asarray(x, dtype=np.float64)
    Nc = p.countries
    a = np.exp(x[..., :Nc] * 2.0 * p.lna_half_width - p.lna_half_width)
    k = p.k_lo + x[..., Nc:] * (p.k_hi - p.k_lo)
    return a, k


def _handles(policy):
    if isinstance(policy, VectorizedDdsg):
        return policy._h, None
    if isinstance(policy, SparseGridFunction):
        return None, policy._h
    raise InvalidArgument("irbc: policy must be a VectorizedDdsg or SparseGridFunction")


def _buf(x, cols: int, name: str):
    if hasattr(x, "data_ptr") and not isinstance(x, np.ndarray):
        import torch

        if x.dtype != torch.float64:
            raise InvalidArgument(f"{name} must be float64")
        t = x.reshape(-1, cols).contiguous()
        return t, t.shape[0]
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1, cols)
    return arr, arr.shape[0]


def _empty(like, shape, dtype=np.float64):
    if isinstance(like, np.ndarray):
        return np.empty(shape, dtype=dtype)
    import torch

    tdt = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
    return torch.empty(shape, dtype=tdt, device=like.device)


def foc_residuals(policy, p: IrbcParameters, a, k, candidate, stream: Optional[int] = None):
    """Residuals [n][pdim] and clamped-successor counts [n] of n states."""
    Nc, pd = p.countries, p.policy_dim()
    a, n = _buf(a, Nc, "a")
    k, nk = _buf(k, Nc, "k")
    cand, nc = _buf(candidate, pd, "candidate")
    if not (n == nk == nc):
        raise InvalidArgument("foc_residuals: state / candidate count mismatch")
    res = _empty(a, (n, pd))
    clamped = _empty(a, (n,), np.int32)
    hd, gd = _handles(policy)
    s, g, t = p._c()
    bad = C.c_int64(-1)
    with _DeviceScope(a, stream) as sh:
        st = N.lib.ddsg_irbc_foc_residuals(hd, gd, C.byref(s), n, _ptr(a), _ptr(k), _ptr(cand), _ptr(res),
                                           _ptr(clamped), C.byref(bad), C.c_void_p(sh))
    _check(st, bad.value)
    return res, clamped


def foc_jacobian(policy, p: IrbcParameters, a, k, z, r0, fd_epsilon: float = 1e-7,
                 stream: Optional[int] = None):
    """Forward-difference Newton matrices jac[n][pdim][pdim] (solver.hpp:129-165;
    SolverConfig::fd_epsilon default 1e-7, solver.hpp:40)."""
    Nc, pd = p.countries, p.policy_dim()
    a, n = _buf(a, Nc, "a")
    k, nk = _buf(k, Nc, "k")
    z, nz = _buf(z, pd, "z")
    r0, nr = _buf(r0, pd, "r0")
    if not (n == nk == nz == nr):
        raise InvalidArgument("foc_jacobian: state count mismatch")
    jac = _empty(a, (n, pd, pd))
    hd, gd = _handles(policy)
    s, g, t = p._c()
    bad = C.c_int64(-1)
    with _DeviceScope(a, stream) as sh:
        st = N.lib.ddsg_irbc_foc_jacobian(hd, gd, C.byref(s), n, _ptr(a), _ptr(k), _ptr(z), _ptr(r0),
                                          float(fd_epsilon), _ptr(jac), C.byref(bad), C.c_void_p(sh))
    _check(st, bad.value)
    return jac


@dataclass
class EulerErrors:
    """solver.hpp:369-373 (+ the clamp count the reference returns through a pointer)."""

    avg_log10: float
    max_log10: float
    samples: np.ndarray
    clamp_count: int = 0


def euler_errors_at(policy, p: IrbcParameters, xs, stream: Optional[int] = None) -> EulerErrors:
    """euler_errors on caller-supplied canonical samples xs[n][2N]."""
    xs, n = _buf(xs, p.state_dim(), "xs")
    if n < 1:
        raise InvalidArgument("euler_errors: n_samples must be >= 1")
    errs = _empty(xs, (n,))
    mean, worst, cl = C.c_double(), C.c_double(), C.c_uint64()
    hd, gd = _handles(policy)
    s, g, t = p._c()
    bad = C.c_int64(-1)
    with _DeviceScope(xs, stream) as sh:
        st = N.lib.ddsg_irbc_euler_errors(hd, gd, C.byref(s), n, _ptr(xs), _ptr(errs), C.byref(mean),
                                          C.byref(worst), C.byref(cl), C.byref(bad), C.c_void_p(sh))
    _check(st, bad.value)
    # solver.hpp:431-432 (host log10, as the reference)
    m, w = mean.value, worst.value
    return EulerErrors(math.log10(m if not (m < 1e-16) else 1e-16), math.log10(w if not (w < 1e-16) else 1e-16),
                       errs, int(cl.value))


def euler_errors(policy, p: IrbcParameters, n_samples: int, seed: int, workers: Optional[int] = None,
                 stream: Optional[int] = None) -> EulerErrors:
    """solver.hpp:377-436: samples from std::mt19937_64(seed) +
    uniform_real_distribution(0,1), drawn up front (``workers`` is accepted for
    signature parity; the result never depends on it)."""
    if n_samples < 1:
        raise InvalidArgument("euler_errors: n_samples must be >= 1")
    xs = uniform_points(seed, n_samples, p.state_dim())
    return euler_errors_at(policy, p, xs, stream)
