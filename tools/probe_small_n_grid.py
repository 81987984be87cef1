"""Device time of small batches on the plain-grid configs (1-3): the latency
a per-point interpolate(x, out) caller sees.  Usage:
python tools/probe_small_n_grid.py <config> n1 n2 ...   -> JSON lines"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import last_eval_stats


def main():
    cid = int(sys.argv[1])
    ns = [int(v) for v in sys.argv[2:]]
    cfg = W.CONFIGS[cid]
    g = W.build_grid(cfg)
    xs = torch.from_numpy(W.points(cfg, n=max(ns))).cuda()
    for n in ns:
        x = xs[:n].contiguous()
        y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
        for _ in range(3):
            g.interpolate(x, out=y)
        dev, wall = [], []
        for _ in range(20):
            torch.cuda.synchronize()
            t = time.perf_counter()
            g.interpolate(x, out=y)
            wall.append(time.perf_counter() - t)
            dev.append(last_eval_stats()[1])
        dev.sort()
        wall.sort()
        print(json.dumps({"config": cid, "n": n, "device_ms_median": dev[len(dev) // 2],
                          "call_us_median": wall[len(wall) // 2] * 1e6}), flush=True)


if __name__ == "__main__":
    main()
