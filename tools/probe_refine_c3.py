"""Config 3 from level 5 to level 6 by one refinement step with GPU residual
hierarchization (refine.py) against the host build at
level 6 (bit-exact node set and surpluses).  Usage: probe_refine_c3.py"""
import dataclasses
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.refine import refine_step

cfg5 = W.CONFIGS[3]
cfg6 = dataclasses.replace(cfg5, max_level=6)
t = time.time()
g = W.build_grid(cfg5)
t_l5 = time.time() - t
f = W.GridTarget(cfg5)
t = time.time()
dev = "--host" not in sys.argv
st = refine_step([g], [cfg5.max_level + cfg5.d - 1], lambda gi, xs: f(xs), dist=None, device=dev)
t_gpu = time.time() - t
t = time.time()
h = W.build_grid(cfg6)
t_host = time.time() - t
k1, s1 = g.nodes()
k2, s2 = h.nodes()
same = np.array_equal(k1, k2) and np.array_equal(s1.view(np.uint64), s2.view(np.uint64))
print(f"L5 host build {t_l5:.1f}s; refine to L6 on the GPU: {t_gpu:.2f}s (new nodes {st.new_nodes}, "
      f"hierarchize {st.hierarchize_s:.2f}s, target {st.target_s:.2f}s); host build at L6 {t_host:.1f}s; "
      f"bit-identical: {same}", flush=True)
