"""Why FAST (FMA) mode cannot be certified by an a-posteriori bound (SURVEY.md
§7 H1), measured on configs 4 and 5.

For each sampled point p and output c:
  E = EXACT evaluation (bit-identical to the reference), F = FAST (one DFMA
  per term, same order), tol = 1e-14 + 1e-12 |E| (the north star);
  A_s[p,c] = sum_t |w_t(p)| |s_t[c]|  (slot s, terms t: the exact abs sum);
  B = 2 (gamma_{n_max+1} + gamma_depth) sum_s |b_s| A_s    (rigorous |F - E| bound:
      both F and E are within (gamma_{n+1} + gamma_depth) sum |b_s| A_s of the
      exact value, n = terms per slot, depth = pairwise tree depth);
  B_cheap = the same with A_s <= W_s M_s[c] (W_s = sum_t |w_t|,
      M_s[c] = max_t |s_t[c]|), the per-slot form SURVEY.md H1 proposes.
An output is "flagged" (needs the exact recompute) when its bound exceeds
tol.  Reported: violations (|F - E| > tol), flagged fractions, and the
cancellation ratio sum_s |b_s row_s| / |y| that makes B large.

Usage (GPU): python tools/probe_fast_bound.py [n_points]   -> one JSON object
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import EXACT, FAST

U = 2.0 ** -53


def gamma(n):
    return n * U / (1 - n * U)


def basis(mode, lv, idx, x):
    """basis_kind / basis_value (basis.hpp:27-54), vectorised over nodes (lv,
    idx) and points x."""
    inv_h = np.ldexp(1.0, lv)
    hat = np.maximum(1.0 - np.abs(x - idx / inv_h) * inv_h, 0.0)
    if mode == 0:
        return hat
    left = np.maximum(2.0 - x * inv_h, 0.0)
    right = np.maximum(2.0 - (1.0 - x) * inv_h, 0.0)
    v = np.where(idx == (1 << lv) - 1, right, hat)
    v = np.where(idx == 1, left, v)
    return np.where(lv == 1, 1.0, v)


def probe(cid, n):
    import torch

    cfg = W.CONFIGS[cid]
    vec, parts = W.build_hdmr(cfg)
    x = W.points(cfg, n=n, seed=99)
    xd = torch.from_numpy(x).cuda()
    vec.set_eval_mode(EXACT)
    e = vec.evaluate_batch(xd).cpu().numpy()
    vec.set_eval_mode(FAST)
    f = vec.evaluate_batch(xd).cpu().numpy()
    vec.set_eval_mode(EXACT)
    tol = 1e-14 + 1e-12 * np.abs(e)
    sum_a = np.zeros_like(e)
    sum_cheap = np.zeros_like(e)
    sum_row = np.zeros_like(e)
    n_max = 1
    active = [(u, b, g) for u, b, g in parts.slots if b != 0]
    for u, b, g in active:
        if g is None:
            r = np.abs(b * parts.f_anchor)[None, :]
            sum_a += r
            sum_cheap += r
            sum_row += r
            continue
        keys, sur = g.nodes()
        lv = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64) + 1
        idx = 2 * (keys.astype(np.int64) - (np.int64(1) << (lv - 1))) + 1
        w = np.ones((n, keys.shape[0]))
        for j, dim in enumerate(u):
            w *= basis(g.boundary_mode, lv[:, j][None, :], idx[:, j][None, :], x[:, dim][:, None])
        n_max = max(n_max, int(np.count_nonzero(w, axis=1).max()))
        sum_a += abs(b) * (np.abs(w) @ np.abs(sur))
        sum_cheap += abs(b) * np.abs(w).sum(axis=1)[:, None] * np.abs(sur).max(axis=0)[None, :]
        sum_row += np.abs(b * (w @ sur))
    depth = int(np.ceil(np.log2(len(active))))
    k = 2 * (gamma(n_max + 1) + gamma(depth))
    bound, cheap = k * sum_a, k * sum_cheap
    err = np.abs(f - e)
    return {
        "config": cfg.name, "points": n, "outputs": int(e.size), "active_slots": len(active),
        "terms_per_slot_max": n_max, "tree_depth": depth,
        "violations": int((err > tol).sum()), "max_err_over_tol": float((err / tol).max()),
        "bit_identical_fraction": float((f.view(np.uint64) == e.view(np.uint64)).mean()),
        "flagged_fraction_exact_abs_sum": float((bound > tol).mean()),
        "flagged_fraction_per_slot_WM": float((cheap > tol).mean()),
        "median_bound_over_tol": float(np.median(bound / tol)),
        "median_cancellation_sum_b_row_over_y": float(np.median(sum_row / np.maximum(np.abs(e), 1e-300))),
    }


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    print(json.dumps({"c4": probe(4, n), "c5": probe(5, n)}))
