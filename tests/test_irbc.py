"""Batched IRBC policy callers against the
reference: refresh_derived / steady_state_lambda / foc_residuals are the
reference's own (oracle/_ref), foc_jacobian and euler_errors the oracle
driver's Eigen-free restatements of solver.hpp:129-165 / 377-436 on top of
the reference's foc_residuals.  Known answers restate test_irbc.cpp and
test_solver.cpp.

Tolerances: the policy values at a given successor state are bit-identical
(EXACT evaluation); successor productivities go through exp/log, which are
CUDA's (<= 1-2 ulp) instead of glibc's, so residuals agree to rounding:
|d| <= 1e-12 (1 + |ref|).  Forward-difference Jacobians divide that by
h = 1e-7 max(|z|, 1e-2): |d| <= 1e-6 (1 + |J|) elementwise, the reference's
own Jacobian test allows 1e-5 (test_solver.cpp:131).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle_lib as O
from paper_2202_06555_b200 import irbc as I
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import DomainError, InvalidArgument

RES_TOL = 1e-12
JAC_TOL = 1e-6


def need_ref():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")


# ------------------------------------------------------------ host (CPU)

@pytest.mark.parametrize("countries", [1, 2, 4, 7, 150])
@pytest.mark.parametrize("variant", [I.SMOOTH, I.NONSMOOTH])
def test_refresh_derived_matches_reference(countries, variant):
    need_ref()
    p = I.make_parameters(countries, variant, gamma_base=0.3)
    rc, g, t, A = O.ref_irbc_refresh(I.IrbcParameters(countries=countries, variant=variant, gamma_base=0.3))
    assert rc == 0
    assert np.array_equal(np.array(p.gamma), g) and np.array_equal(np.array(p.tau), t) and p.A == A
    q = I.make_identical_gamma_parameters(countries, variant, 0.5)
    assert q.gamma == [0.5] * countries
    assert I.steady_state_lambda(p) == O.ref_irbc_steady_lambda(p)
    assert I.steady_state_lambda(q) == O.ref_irbc_steady_lambda(q)


def test_calibration_known_answers():
    # test_irbc.cpp:28-52
    p = I.make_parameters(4)
    assert abs(p.A - (1.0 - 0.99 * 0.99) / (0.36 * 0.99)) <= 1e-15
    assert np.allclose(p.gamma, [0.25, 0.5, 0.75, 1.0], rtol=0, atol=1e-15)
    for j in range(4):
        assert abs(p.tau[j] - p.A ** (1.0 / p.gamma[j])) <= 1e-15
    assert abs(1.0 - p.beta * (p.alpha * p.A + 1.0 - p.delta)) < 1e-12
    assert I.make_parameters(1).gamma == [0.25]
    lam = I.steady_state_lambda(p)
    assert abs(sum(p.A * lam ** -g for g in p.gamma) - 4.0 * (p.A - p.delta)) <= 1e-10


@pytest.mark.parametrize("field,value,msg", [
    ("beta", 1.5, "beta in (0,1)"), ("delta", 0.0, "delta in (0,1)"), ("alpha", 1.0, "alpha in (0,1)"),
    ("sigma", -1.0, "sigma must be >= 0"), ("rho_a", 1.0, "rho_a in [0,1)"), ("phi_adj", -0.1, "phi_adj"),
    ("k_lo", 0.0, "capital box"), ("lna_half_width", 0.0, "lna_half_width"), ("countries", 0, "countries"),
])
def test_refresh_derived_rejects_bad_parameters(field, value, msg):
    p = I.IrbcParameters(countries=3)
    setattr(p, field, value)
    with pytest.raises(InvalidArgument, match=msg.replace("(", r"\(").replace(")", r"\)").replace("[", r"\[")):
        I.refresh_derived(p)
    bad = I.IrbcParameters(countries=2, gamma=[0.5, -1.0])
    with pytest.raises(InvalidArgument, match="gamma_j must be > 0"):
        I.refresh_derived(bad)


def test_shock_quadrature_layout():
    nodes, w = I.make_shock_quadrature(3)
    assert nodes.shape == (8, 4) and np.all(w == 1.0 / 8.0)
    assert nodes[0, 0] == math.sqrt(4.0) and nodes[1, 0] == -2.0 and nodes[7, 3] == -2.0
    assert np.count_nonzero(nodes) == 8
    with pytest.raises(InvalidArgument):
        I.make_shock_quadrature(0)


def test_policy_target_shapes():
    t = W.IrbcPolicyTarget(3, nonsmooth=True, n_pairs=4, lam0=1.5)
    y = t(np.full((2, 6), 0.5))
    assert y.shape == (2, 7)
    # at the center: k' = (1-delta) k + delta k = k = 1, mu = 0, lambda = lam0
    assert np.allclose(y[:, :3], 1.0) and np.all(y[:, 3:6] == 0.0) and np.all(y[:, 6] == 1.5)
    s = W.IrbcPolicyTarget(2, steady=True, lam0=2.0)
    x = np.array([[0.1, 0.9, 0.25, 0.75]])
    assert np.array_equal(s(x), np.array([[0.75, 1.25, 2.0]]))


# ------------------------------------------------------------ GPU parity

def ref_policy_of(policy, parts=None):
    """The same bits as a reference policy (from_nodes / from_parts)."""
    if parts is None:
        keys, sur = policy.nodes()
        return O.ref_from_nodes(policy.dim, policy.out_dim, policy.boundary_mode, policy.max_level,
                                policy.eps_gamma, keys, sur)
    grids = []
    for u, b, g in parts.slots:
        if g is None:
            grids.append(None)
        else:
            keys, sur = g.nodes()
            grids.append(O.ref_from_nodes(len(u), parts.m, g.boundary_mode, g.max_level, g.eps_gamma, keys, sur))
    return O.RefHdmr(parts.d, parts.m, parts.f_anchor, [(u, b) for u, b, _ in parts.slots], grids)


def random_states(p, n, seed, box=1.0):
    rng = np.random.default_rng(seed)
    x = 0.5 + box * (rng.random((n, p.state_dim())) - 0.5)
    a, k = I.from_canonical(x, p)
    return x, a, k


def close(got, want, tol):
    return np.abs(got - want) <= tol * (1.0 + np.abs(want))


@pytest.fixture(scope="module")
def smooth2():
    p = I.make_parameters(2, I.SMOOTH)
    t = W.IrbcPolicyTarget(2, n_pairs=2, lam0=I.steady_state_lambda(p))
    vec, parts = W.build_policy_hdmr(t, 6, 4)
    return p, t, vec, parts, ref_policy_of(vec, parts)


@pytest.fixture(scope="module")
def nonsmooth3():
    p = I.make_parameters(3, I.NONSMOOTH)
    t = W.IrbcPolicyTarget(3, nonsmooth=True, n_pairs=4, lam0=I.steady_state_lambda(p))
    vec, parts = W.build_policy_hdmr(t, 6, 4)
    return p, t, vec, parts, ref_policy_of(vec, parts)


@pytest.fixture(scope="module")
def grid4():
    p = I.make_parameters(4, I.SMOOTH)
    t = W.IrbcPolicyTarget(4, lam0=I.steady_state_lambda(p))
    g = W.build_policy_grid(t, 4)
    return p, t, g, None, ref_policy_of(g)


CASES = ["smooth2", "nonsmooth3", "grid4"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_policy_evaluation_is_bitwise_reference(case, request):
    """The policies are adaptive builds stored in several runs; the batched
    evaluation underneath the callers is the reference's, bit for bit."""
    need_ref()
    p, t, pol, parts, rpol = request.getfixturevalue(case)
    x, _, _ = random_states(p, 500, 21)
    if parts is None:
        got = pol.interpolate(x)
        rc, want = rpol.eval(x, p.policy_dim())
    else:
        assert pol.uses_slot_kernel()
        got = pol.evaluate_batch(x)
        rc, want = rpol.eval(x)
    assert rc == 0
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_foc_residuals_match_reference(case, request):
    need_ref()
    p, t, pol, parts, rpol = request.getfixturevalue(case)
    # states over the whole box, candidates = target policy perturbed, a few
    # pushed out of the box so successors clamp
    x, a, k = random_states(p, 97, 11)
    cand = t(x) * (1.0 + 0.02 * (np.random.default_rng(3).random((97, p.policy_dim())) - 0.5))
    cand[:5, 0] = p.k_hi + 0.05
    cand[5:8, 0] = p.k_lo - 0.05
    res, cl = I.foc_residuals(pol, p, a, k, cand)
    rres, rcl = O.ref_irbc_foc_residuals(rpol, p, a, k, cand)
    assert np.array_equal(cl, rcl)
    assert np.all(cl[:8] > 0)
    ok = close(res, rres, RES_TOL)
    assert ok.all(), np.abs(res - rres).max()


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_foc_jacobian_matches_reference(case, request):
    need_ref()
    p, t, pol, parts, rpol = request.getfixturevalue(case)
    x, a, k = random_states(p, 13, 5, box=0.7)
    z = t(x)
    if p.variant == I.NONSMOOTH:
        z[:3, p.countries] = 0.0  # FB corner rows: mu = 0, slack = 0 handled analytically
        z[:3, 0] = (1.0 - p.delta) * k[:3, 0]
    r0, _ = O.ref_irbc_foc_residuals(rpol, p, a, k, z)
    jac = I.foc_jacobian(pol, p, a, k, z, r0)
    rjac = O.ref_irbc_foc_jacobian(rpol, p, a, k, z, r0)
    ok = close(jac, rjac, JAC_TOL)
    assert ok.all(), np.abs(jac - rjac).max()
    if p.variant == I.NONSMOOTH:
        N = p.countries
        assert np.array_equal(jac[:, N:2 * N, :], rjac[:, N:2 * N, :])  # analytic rows: exact


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_euler_errors_match_reference(case, request):
    need_ref()
    p, t, pol, parts, rpol = request.getfixturevalue(case)
    e = I.euler_errors(pol, p, 300, 99)
    xs = O.port_uniform_points(99, 300, p.state_dim())
    errs, mean, worst, cl = O.ref_irbc_euler_errors(rpol, p, xs, workers=4)
    assert e.clamp_count == cl
    assert close(e.samples, errs, RES_TOL).all(), np.abs(e.samples - errs).max()
    assert abs(e.avg_log10 - math.log10(max(mean, 1e-16))) <= 1e-11
    assert abs(e.max_log10 - math.log10(max(worst, 1e-16))) <= 1e-11
    # determinism (test_solver.cpp:180-195)
    e2 = I.euler_errors(pol, p, 300, 99)
    assert np.array_equal(e.samples, e2.samples) and e.avg_log10 == e2.avg_log10


# ------------------------------------------------ known answers (reference)

def steady_grid(p, lam):
    t = W.IrbcPolicyTarget(p.countries, nonsmooth=p.variant == I.NONSMOOTH, steady=True, lam0=lam,
                           k_lo=p.k_lo, k_hi=p.k_hi, lna_half_width=p.lna_half_width)
    return W.build_policy_grid(t, 2)


@pytest.mark.gpu
def test_smooth_residuals_vanish_at_steady_state():
    # test_irbc.cpp:189-206
    p = I.make_identical_gamma_parameters(2, I.SMOOTH, 0.25)
    p.sigma = 0.0
    I.refresh_derived(p)
    lam = I.steady_state_lambda(p)
    assert abs(lam - (1.0 - p.delta / p.A) ** (-1.0 / 0.25)) <= 1e-10
    res, _ = I.foc_residuals(steady_grid(p, lam), p, [[1.0, 1.0]], [[1.0, 1.0]], [[1.0, 1.0, lam]])
    assert np.all(np.abs(res) < 1e-10)


@pytest.mark.gpu
def test_bare_euler_row_with_phi_zero():
    # test_irbc.cpp:208-236: phi = 0, k' = k
    p = I.make_parameters(2, I.SMOOTH)
    p.phi_adj = 0.0
    I.refresh_derived(p)
    lam_next = I.steady_state_lambda(p)
    a, k = np.array([1.05, 0.93]), np.array([1.2, 0.8])
    res, _ = I.foc_residuals(steady_grid(p, lam_next), p, [a], [k], [[1.2, 0.8, 1.5]])
    nodes, w = I.make_shock_quadrature(2)
    for j in range(2):
        expec = 0.0
        for q in range(nodes.shape[0]):
            an = math.exp(p.rho_a * math.log(a[j]) + p.sigma * (nodes[q, j] + nodes[q, 2]))
            expec += w[q] * lam_next * (an * p.A * p.alpha * k[j] ** (p.alpha - 1.0) + 1.0 - p.delta)
        assert abs(res[0, j] - (1.5 - p.beta * expec)) <= 1e-12


@pytest.mark.gpu
def test_nonsmooth_rows_at_slack_and_binding():
    # test_irbc.cpp:247-275
    p = I.make_identical_gamma_parameters(2, I.NONSMOOTH, 0.25)
    p.sigma = 0.0
    I.refresh_derived(p)
    lam = I.steady_state_lambda(p)
    pol = steady_grid(p, lam)
    res, _ = I.foc_residuals(pol, p, [[1.0, 1.0]], [[1.0, 1.0]], [[1.0, 1.0, 0.0, 0.0, lam]])
    assert np.all(np.abs(res) < 1e-10)
    res, _ = I.foc_residuals(pol, p, [[1.0, 1.0]], [[1.0, 1.0]], [[1.0 - p.delta, 1.0, 0.2, 0.0, lam]])
    assert abs(res[0, 2]) < 1e-12


@pytest.mark.gpu
def test_clamped_successors_are_counted():
    # test_irbc.cpp:277-292
    p = I.make_parameters(2, I.SMOOTH)
    pol = steady_grid(p, I.steady_state_lambda(p))
    _, cl = I.foc_residuals(pol, p, [[1.0, 1.0]], [[1.49, 1.0]], [[1.52, 1.0, 1.5]])
    assert cl[0] == 6


@pytest.mark.gpu
def test_euler_errors_degenerate_box_is_exact():
    # test_solver.cpp:170-196
    p = I.make_identical_gamma_parameters(2, I.SMOOTH, 0.25)
    p.sigma = 0.0
    p.k_lo, p.k_hi, p.lna_half_width = 1.0 - 5e-11, 1.0 + 5e-11, 5e-11
    I.refresh_derived(p)
    pol = steady_grid(p, I.steady_state_lambda(p))
    e1 = I.euler_errors(pol, p, 500, 99)
    assert e1.avg_log10 < -8.0 and e1.max_log10 < -8.0
    e2 = I.euler_errors(pol, p, 500, 99, workers=4)
    assert np.array_equal(e1.samples, e2.samples) and e1.max_log10 == e2.max_log10
    doubled = np.concatenate([e1.samples, e1.samples])
    assert doubled.max() == e1.samples.max()


@pytest.mark.gpu
def test_jacobian_against_central_differences(smooth2):
    # test_solver.cpp:95-133: forward differences vs central differences, 1e-5
    p, t, pol, parts, _ = smooth2
    rng = np.random.default_rng(23)
    n, pd = 40, p.policy_dim()
    x = rng.uniform(0.15, 0.85, (n, p.state_dim()))
    a, k = I.from_canonical(x, p)
    lam = I.steady_state_lambda(p)
    z = np.concatenate([k, lam * (0.9 + 0.2 * rng.random((n, 1)))], axis=1)
    r0, _ = I.foc_residuals(pol, p, a, k, z)
    jac = I.foc_jacobian(pol, p, a, k, z, r0)
    cd = np.empty_like(jac)
    for c in range(pd):
        h = 1e-5 * np.maximum(np.abs(z[:, c]), 1e-2)
        zp, zm = z.copy(), z.copy()
        zp[:, c] += h
        zm[:, c] -= h
        rp, _ = I.foc_residuals(pol, p, a, k, zp)
        rm, _ = I.foc_residuals(pol, p, a, k, zm)
        cd[:, :, c] = (rp - rm) / (2.0 * h[:, None])
    for i in range(n):
        assert np.linalg.norm(jac[i] - cd[i]) / np.linalg.norm(cd[i]) <= 1e-5


# ------------------------------------------------------------ boundaries

@pytest.mark.gpu
def test_device_tensors_match_host(smooth2):
    import torch

    p, t, pol, _, _ = smooth2
    x, a, k = random_states(p, 33, 8)
    cand = t(x)
    res_h, cl_h = I.foc_residuals(pol, p, a, k, cand)
    dev = [torch.from_numpy(v).cuda() for v in (a, k, cand)]
    res_d, cl_d = I.foc_residuals(pol, p, *dev)
    assert np.array_equal(res_h, res_d.cpu().numpy()) and np.array_equal(cl_h, cl_d.cpu().numpy())


@pytest.mark.gpu
def test_nan_candidate_is_a_domain_error_with_lowest_state(smooth2):
    p, t, pol, _, _ = smooth2
    x, a, k = random_states(p, 20, 9)
    cand = t(x)
    cand[13, 1] = np.nan
    cand[17, 0] = np.nan
    with pytest.raises(DomainError) as ei:
        I.foc_residuals(pol, p, a, k, cand)
    assert ei.value.task_id == 13


@pytest.mark.gpu
def test_policy_dimension_mismatch_is_rejected(smooth2, grid4):
    p, _, pol, _, _ = smooth2
    p4 = grid4[0]
    with pytest.raises(InvalidArgument, match="policy dimensions"):
        I.foc_residuals(pol, p4, np.ones((1, 4)), np.ones((1, 4)), np.ones((1, 5)))
    with pytest.raises(InvalidArgument):
        I.euler_errors(pol, p, 0, 1)


@pytest.mark.gpu
def test_empty_batch(smooth2):
    p, _, pol, _, _ = smooth2
    res, cl = I.foc_residuals(pol, p, np.ones((0, 2)), np.ones((0, 2)), np.ones((0, 3)))
    assert res.shape == (0, 3) and cl.shape == (0,)
