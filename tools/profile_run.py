"""One evaluation of a config on device-resident points (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2202_06555_b200 import workloads as W

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = W.CONFIGS[cid]
obj = W.build_grid(cfg) if cfg.kind == "grid" else W.build_hdmr(cfg)[0]
x = torch.from_numpy(W.points(cfg, n=n)).cuda()
y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
ev = obj.interpolate if cfg.kind == "grid" else obj.evaluate_batch
for _ in range(reps):
    ev(x, out=y)
torch.cuda.synchronize()
print("done", float(y[0, 0]))
