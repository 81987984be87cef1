"""Quick timing probe of the evaluation kernels on configs (device-resident inputs)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import last_eval_stats, EXACT, FAST

def run(cid, n, modes=(EXACT,)):
    cfg = W.CONFIGS[cid]
    t = time.time()
    obj = W.build_grid(cfg) if cfg.kind == "grid" else W.build_hdmr(cfg)[0]
    tb = time.time() - t
    x = torch.from_numpy(W.points(cfg, n=n)).cuda()
    y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
    ev = obj.interpolate if cfg.kind == "grid" else obj.evaluate_batch
    nnz, _ = obj.support(x[: min(n, 4096)].cpu().numpy())
    for mode in modes:
        obj.set_eval_mode(mode)
        ev(x, out=y)
        ms = []
        for _ in range(3):
            ev(x, out=y)
            ms.append(last_eval_stats()[2])
        kms = min(ms)
        flops = 2.0 * cfg.m * nnz.mean() * n
        print(f"config{cid} n={n} mode={'exact' if mode==EXACT else 'fast'} build={tb:.1f}s kernel={kms:.2f}ms "
              f"evals/s={n*cfg.m/kms*1e3:.3e} nnz/pt={nnz.mean():.1f} TFLOP/s={flops/kms/1e9:.2f}", flush=True)

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        cid, n = spec.split(":")
        run(int(cid), int(n), (EXACT, FAST))
