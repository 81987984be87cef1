"""Term-parallel plain kernel (plain_terms_kernel) against the serial walk
(plain_kernel) on config 1 and small random single-output grids: kernel time
per batch size and bitwise equality of the outputs.  Each form runs in a
child process (DDSG_PLAIN_TERMS is read once per process).

Usage: python tools/probe_plain_terms.py [n ...]  -> JSON lines
"""
import hashlib, json, os, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SIZES = [512, 4096, 65536, 1 << 18, 1 << 19]

CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import last_eval_stats, SparseGridFunction
cfg = W.CONFIGS[1]
g = W.build_grid(cfg)
out = {}
for n in %r:
    x = torch.from_numpy(W.points(cfg, n=n)).cuda()
    y = torch.empty((n, cfg.m), dtype=torch.float64, device="cuda")
    g.interpolate(x, out=y)
    ms = []
    for _ in range(5):
        g.interpolate(x, out=y)
        ms.append(last_eval_stats()[2])
    out[str(n)] = {"kernel_us": min(ms) * 1e3, "sha": hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]}
print(json.dumps(out))
"""


def child(terms: int):
    env = dict(os.environ, DDSG_PLAIN_TERMS=str(terms))
    r = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), SIZES)], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        raise SystemExit(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    if len(sys.argv) > 1:
        SIZES = [int(v) for v in sys.argv[1:]]
    a, b = child(0), child(1)
    for n in SIZES:
        ra, rb = a[str(n)], b[str(n)]
        print(json.dumps({"config": 1, "points": n, "serial_walk_us": round(ra["kernel_us"], 2),
                          "term_parallel_us": round(rb["kernel_us"], 2),
                          "speedup": round(ra["kernel_us"] / rb["kernel_us"], 2),
                          "bit_identical": ra["sha"] == rb["sha"]}))
