"""bench.py's JSON contract, checked on the CPU through the reference arm
(which runs the reference's own evaluator from oracle/_ref, no GPU), and the
graft entry points' surface."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

import oracle_lib as O

ROOT = Path(__file__).resolve().parent.parent


def run_bench(*args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=str(ROOT), env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    d = run_bench("--impl", "reference", "--config", "4", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "evals/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "config4_hdmr_d100"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the reference arm maps only oracle/_ref: no product library in its process
    assert d["repo_libraries_loaded"] and all(p.startswith("oracle/_ref/") for p in d["repo_libraries_loaded"])


def test_reference_arm_builds_the_same_program():
    """oracle/ref_workload.py (reference build, reference b lattice, targets
    linked into oracle/_ref, reference point generator) reproduces the
    product's config-4 program: same family and b, same anchor values, same
    node bits per cut, and the same blocked point stream."""
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    import numpy as np

    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_workload as RW
    from helpers import bits
    from paper_2202_06555_b200 import workloads as W
    from paper_2202_06555_b200.ddsg import uniform_point_blocks

    cfg = RW.configs()[4]
    lib = RW.use_library(O.REF_PATH)
    ref, fa, fam, b = RW.build_hdmr(cfg, lib)
    parts = W.build_hdmr_parts(W.CONFIGS[4])
    assert [u for u, _, _ in parts.slots] == fam
    assert [bu for _, bu, _ in parts.slots] == b
    assert np.array_equal(bits(parts.f_anchor), bits(fa))
    for (u, bu, g), rg in zip(parts.slots, ref._keep):
        if g is None:
            assert rg is None
            continue
        k1, s1 = g.nodes()
        k2, s2 = rg.nodes(len(u), cfg.m)
        assert np.array_equal(k1, k2) and np.array_equal(bits(s1), bits(s2))
    first, n = RW.BLOCK_POINTS - 5, 2 * RW.BLOCK_POINTS + 9
    x_ref = RW.points(lib, cfg, first, n)
    x_ours = uniform_point_blocks(cfg.seed, RW.BLOCK_POINTS, first, n, cfg.d)
    assert np.array_equal(bits(x_ref), bits(x_ours))
    # a shard is the same points whatever the split
    a = uniform_point_blocks(cfg.seed, RW.BLOCK_POINTS, 0, 3000, cfg.d)
    b2 = np.concatenate([uniform_point_blocks(cfg.seed, RW.BLOCK_POINTS, 0, 1234, cfg.d),
                         uniform_point_blocks(cfg.seed, RW.BLOCK_POINTS, 1234, 3000 - 1234, cfg.d)])
    assert np.array_equal(bits(a), bits(b2))


def test_reference_arm_non_zero_rank_is_silent():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "4"],
                       capture_output=True, text=True, timeout=300, cwd=str(ROOT),
                       env={**os.environ, "RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_graft_entry_surface():
    sys.path.insert(0, str(ROOT))
    import __graft_entry__ as g

    assert callable(g.build) and callable(g.smoke)


@pytest.mark.gpu
def test_bench_default_line_on_gpu():
    d = run_bench("--steps", "3", "--warmup", "3", "--points", "65536", "--no-cpu-baseline", "--no-refine",
                  timeout=900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    rf = d["roofline"]
    assert rf["bound"] in ("fp64", "hbm", "tensor") and 0 < rf["frac"] < 1 and rf["peak"] > 0
    # the resource that binds the slot kernel: the shared-memory gather ceiling
    br = rf["binding_resource"]
    assert 0 < br["frac"] < 1 and br["peak"] > 0 and abs(br["achieved"] - rf["achieved"]) < 1e-9
    assert br["peak"] < rf["peak"]  # 16 doubles/clk/SM is below the DFMA rate


@pytest.mark.gpu
def test_bench_parity_field_on_gpu():
    """The bench line carries a bit-exact check of its own timed inputs
    against the reference (oracle/_ref, the reference's own grid build)."""
    d = run_bench("--config", "4", "--steps", "2", "--warmup", "3", "--points", "65536", "--cpu-seconds", "1",
                  timeout=900)
    p = d["parity"]
    assert p["points"] == 4096 and p["bit_identical_points"] == 4096 and p["outputs_outside_tolerance"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] > 0


@pytest.mark.gpu
def test_bench_under_torchrun_nccl_one_rank():
    """The multi-GPU launch path on one GPU: torchrun, a one-rank NCCL group
    (DDSG_BENCH_FORCE_DIST=1), the refinement's surplus all-gather over NCCL,
    then the timed evaluation and the usual JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    e = dict(os.environ, DDSG_BENCH_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--gpus", "1", "--steps", "2", "--warmup", "3", "--points", "65536", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0
    rf = d["refinement"]
    # the native step all-gathered over torch's NCCL communicator, and it had work to do
    assert "ncclAllGather" in rf["collective"] and rf["build"].startswith("rank 0 builds")
    assert rf["new_nodes"] > 0 and rf["rounds"] > 0
    assert rf["allgather_bytes"] == rf["new_nodes"] * d["config"]["m"] * 8
    assert d["parity"] is None or d["parity"]["bit_identical_points"] == d["parity"]["points"]
