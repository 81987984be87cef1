"""Speed of the generic HDMR kernel (the fallback for programs outside the
slot kernel's limits): configs 4 and 5 forced onto it
(DDSG_SLOT_KERNEL=0 vs default), and an order-3 decomposition (k_max = 3:
all 1-d cuts, pairs and triples of 8 dims of config 4's target) that only
the generic kernel runs.  Bit-exactness of every variant is checked against
the slot kernel / the oracle by the GPU tests; this only times.

Usage: [DDSG_SLOT_KERNEL=0] python tools/probe_generic.py   -> JSON lines
"""
import itertools
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import VectorizedDdsg, last_eval_stats


def timed(vec, x, m, nnz_pp):
    y = torch.empty((x.shape[0], m), dtype=torch.float64, device="cuda")
    vec.evaluate_batch(x, out=y)
    ms = []
    for _ in range(3):
        vec.evaluate_batch(x, out=y)
        ms.append(last_eval_stats()[1])
    t = min(ms)
    return {"ms": t, "evals_per_s": x.shape[0] * m / t * 1e3, "tflops_2m_nnz": 2 * m * nnz_pp * x.shape[0] / t / 1e9}


def main():
    tag = "generic" if os.environ.get("DDSG_SLOT_KERNEL") == "0" else "default"
    for cid, n in ((4, 1 << 18), (5, 1 << 16)):
        cfg = W.CONFIGS[cid]
        vec = W.build_hdmr(cfg)[0]
        x = torch.from_numpy(W.points(cfg, n=n)).cuda()
        nnz, _ = vec.support(x[:2048].cpu().numpy())
        r = timed(vec, x, cfg.m, float(nnz.mean()))
        print(json.dumps({"program": cfg.name, "kernel": "slot" if vec.uses_slot_kernel() else "generic",
                          "switch": tag, "points": n, **r}), flush=True)
    # order 3: dims 0..7 of config 4's target, every 1-, 2- and 3-subset
    cfg = W.CONFIGS[4]
    d = cfg.d
    dims8 = range(8)
    fam = [()] + [(k,) for k in range(d)] + list(itertools.combinations(dims8, 2)) + list(itertools.combinations(dims8, 3))
    fam = sorted(fam, key=lambda u: (len(u), u))
    b = W.telescoping_b(fam)
    parts = W.build_hdmr_parts(cfg, build_grids=False)
    grids = {}
    for u in fam:
        if u:
            lvl = {1: 6, 2: 4, 3: 3}[len(u)]
            grids[u] = W.build_cut_grid(cfg, u, lvl, 1e-6)
    slots = [(u, bu, grids.get(u)) for u, bu in zip(fam, b)]
    vec = VectorizedDdsg.compile(d, cfg.m, parts.f_anchor, slots)
    x = torch.from_numpy(W.points(cfg, n=1 << 16)).cuda()
    nnz, _ = vec.support(x[:2048].cpu().numpy())
    r = timed(vec, x, cfg.m, float(nnz.mean()))
    print(json.dumps({"program": "order3_d100_8dims", "slots": len(slots), "kernel": "slot" if vec.uses_slot_kernel()
                      else "generic", "switch": tag, "points": 1 << 16, "nnz_per_point": float(nnz.mean()), **r}),
          flush=True)


if __name__ == "__main__":
    main()
