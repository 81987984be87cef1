import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import oracle_lib as O
from paper_2202_06555_b200 import irbc as I, workloads as W
from test_irbc import ref_policy_of, random_states
for N, ns in [(2, False), (3, True)]:
    p = I.make_parameters(N, I.NONSMOOTH if ns else I.SMOOTH)
    t = W.IrbcPolicyTarget(N, nonsmooth=ns, n_pairs=2*N, lam0=I.steady_state_lambda(p))
    vec, parts = W.build_policy_hdmr(t, 6, 4)
    rv = ref_policy_of(vec, parts)
    x, a, k = random_states(p, 2000, 1)
    z = t(x)
    res, cl = I.foc_residuals(vec, p, a, k, z)
    rres, rcl = O.ref_irbc_foc_residuals(rv, p, a, k, z)
    d = np.abs(res - rres)
    print(N, ns, "residual bit-equal frac", np.mean(res == rres), "max abs", d.max(), "max rel", (d/(1+np.abs(rres))).max())
    jac = I.foc_jacobian(vec, p, a[:50], k[:50], z[:50], rres[:50])
    rj = O.ref_irbc_foc_jacobian(rv, p, a[:50], k[:50], z[:50], rres[:50])
    d = np.abs(jac - rj)
    print("  jac bit-equal frac", np.mean(jac == rj), "max abs", d.max(), "max rel", (d/(1+np.abs(rj))).max())
