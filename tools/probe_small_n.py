"""Device-resident evaluation time of small batches on config 4/5 programs:
the small-batch (slot-parallel) path against the slot kernel.

Usage: DDSG_SMALL_BATCH=<threshold> python tools/probe_small_n.py <config> n1 n2 ...
(DDSG_SMALL_BATCH=0 forces the slot kernel).  Prints one JSON line per n.
"""
import json
import os
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
    vec = W.build_hdmr(cfg)[0]
    xs = torch.from_numpy(W.points(cfg, n=max(ns))).cuda()
    for n in ns:
        x = xs[:n].contiguous()
        y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
        for _ in range(5):
            vec.evaluate_batch(x, out=y)
        dev, wall = [], []
        for _ in range(50):
            torch.cuda.synchronize()
            t = time.perf_counter()
            vec.evaluate_batch(x, out=y)
            wall.append(time.perf_counter() - t)
            dev.append(last_eval_stats()[1])
        wall.sort()
        dev.sort()
        print(json.dumps({"config": cid, "n": n, "small_batch": os.environ.get("DDSG_SMALL_BATCH", "default"),
                          "device_ms_median": dev[len(dev) // 2], "call_us_median": wall[len(wall) // 2] * 1e6}),
              flush=True)


if __name__ == "__main__":
    main()
