"""Probe: does a spatial (Morton) ordering of the query points speed up the
plain-grid kernel?  Times configs 2/3 with points in seeded random order and
in Morton order (same points, device-resident)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import EXACT, last_eval_stats


def morton(x, bits):
    n, d = x.shape
    q = np.minimum((x * (1 << bits)).astype(np.uint64), (1 << bits) - 1)
    key = np.zeros(n, dtype=np.uint64)
    for b in range(bits - 1, -1, -1):
        for k in range(d):
            key = (key << np.uint64(1)) | ((q[:, k] >> np.uint64(b)) & np.uint64(1))
    return key


def run(cid, n):
    cfg = W.CONFIGS[cid]
    obj = W.build_grid(cfg)
    xr = W.points(cfg, n=n)
    bits = max(1, 63 // cfg.d)
    xs = xr[np.argsort(morton(xr, bits), kind="stable")]
    nnz, _ = obj.support(xr[:4096])
    obj.set_eval_mode(EXACT)
    for name, xx in (("random", xr), ("morton", xs)):
        x = torch.from_numpy(np.ascontiguousarray(xx)).cuda()
        y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
        obj.interpolate(x, out=y)
        ms = []
        for _ in range(3):
            obj.interpolate(x, out=y)
            ms.append(last_eval_stats()[2])
        kms = min(ms)
        flops = 2.0 * cfg.m * nnz.mean() * n
        print(f"config{cid} n={n} {name}: kernel={kms:.2f} ms TFLOP/s={flops / kms / 1e9:.2f}", flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        cid, n = spec.split(":")
        run(int(cid), int(n))
