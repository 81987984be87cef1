"""Config 3's target at a higher level cap: build time, nodes, nnz per point and
GPU throughput (EXACT, device-resident points).  Usage: probe_c3_level.py L n"""
import dataclasses
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import last_eval_stats

L, n = int(sys.argv[1]), int(sys.argv[2])
cfg = dataclasses.replace(W.CONFIGS[3], max_level=L)
t = time.time()
g = W.build_grid(cfg)
tb = time.time() - t
x = torch.from_numpy(W.points(cfg, n=n)).cuda()
y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
nnz, _ = g.support(x[:4096].cpu().numpy())
g.interpolate(x, out=y)
ms = []
for _ in range(3):
    g.interpolate(x, out=y)
    ms.append(last_eval_stats()[2])
kms = min(ms)
print(f"config3 L={L} nodes={g.size()} build={tb:.1f}s n={n} kernel={kms:.2f}ms nnz/pt={nnz.mean():.1f} "
      f"evals/s={n * cfg.m / kms * 1e3:.3e} TFLOP/s={2 * cfg.m * nnz.mean() * n / kms / 1e9:.2f}", flush=True)
