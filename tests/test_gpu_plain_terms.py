"""GPU parity of the term-parallel plain kernel (plain_terms_kernel,
csrc/plain.cu): small single-output grids, batches of a few waves.  It must
equal the CPU oracle bit for bit (sparse_grid.hpp:111-128) and the serial
subspace walk (plain_kernel, DDSG_PLAIN_TERMS=0 in a child process)."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from helpers import bits, int_ctx, wl
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import MODIFIED_LINEAR, ZERO_BOUNDARY, DomainError, SparseGridFunction, uniform_points

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

EDGES = np.array([0.0, 1.0, 0.5, 0.25, 0.75, 0.125, 0.875, 1 - 2**-53, 2**-30, 2**-4, 5e-324, 1e-310, 2.0**-1022,
                  2**-60])


def _grid(mode: int, d: int, level: int, eps: float) -> SparseGridFunction:
    keep, ctx = int_ctx(d)
    return SparseGridFunction.build(wl("wl_coupled"), d, 1, level, eps, mode, ctx=ctx)


def _points(d: int, n: int, seed: int) -> np.ndarray:
    x = uniform_points(seed, n, d)
    rng = np.random.default_rng(seed)
    k = min(n // 2, 400)
    x[:k] = EDGES[rng.integers(0, len(EDGES), size=(k, d))]
    return x


def _oracle(g: SparseGridFunction, x):
    keys, sur = g.nodes()
    rc, y, _ = O.port_grid_eval(g.dim, g.out_dim, g.boundary_mode, keys, sur, x)
    assert rc == 0
    return y


@pytest.mark.parametrize("mode", [ZERO_BOUNDARY, MODIFIED_LINEAR])
@pytest.mark.parametrize("d,level,eps", [(1, 7, 0.0), (3, 6, 1e-3), (4, 5, 0.0), (7, 3, 0.0)])
def test_term_parallel_equals_oracle(mode, d, level, eps):
    """Full and adaptive (slab lookups) grids, both boundary modes, cell
    boundaries / ends / subnormal coordinates, ragged batch sizes (300..3,077
    points: beyond the small-batch path, below the Morton-sort threshold)."""
    g = _grid(mode, d, level, eps)
    for n in (300, 1025, 3077):
        x = _points(d, n, 40 + n)
        assert np.array_equal(bits(g.interpolate(x)), bits(_oracle(g, x)))


def test_config1_term_parallel_equals_oracle():
    cfg = W.CONFIGS[1]
    g = W.build_grid(cfg)
    x = W.points(cfg, n=cfg.n_points)
    y = g.interpolate(x)
    assert np.array_equal(bits(y[:6000]), bits(_oracle(g, x[:6000])))


def test_term_parallel_domain_error_lowest_index():
    g = _grid(ZERO_BOUNDARY, 3, 5, 0.0)
    x = _points(3, 2000, 9)
    x[1500, 1] = -1e-300
    x[777, 2] = 1.0 + 1e-12
    x[1999, 0] = np.nan
    with pytest.raises(DomainError) as ei:
        g.interpolate(x)
    assert ei.value.task_id == 777


_CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np
from test_gpu_plain_terms import _grid, _points
from paper_2202_06555_b200.ddsg import EXACT, FAST
out = {}
for mode in (0, 1):
    for d, level, eps in ((2, 8, 1e-4), (4, 5, 0.0), (4, 6, 1e-3)):
        g = _grid(mode, d, level, eps)
        for n in (257, 2049, 40000):
            for em in (EXACT, FAST):
                g.set_eval_mode(em)
                y = g.interpolate(_points(d, n, 3 * n + d))
                out[f"{mode}-{d}-{level}-{n}-{em}"] = hashlib.sha256(np.ascontiguousarray(y).tobytes()).hexdigest()
print(json.dumps(out))
"""


def test_term_parallel_equals_serial_walk():
    """The same grids and points in two child processes: term-parallel form
    (default) and serial walk (DDSG_PLAIN_TERMS=0), EXACT and FAST; d <= 4, so
    40,000 points stay unsorted and take the term-parallel kernel too."""
    res = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", _CHILD, str(ROOT)], env={**os.environ, "DDSG_PLAIN_TERMS": v},
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[0] == res[1] and len(res[0]) == 36
