#!/usr/bin/env python
"""bench.py — batched DDSG interpolant evaluation on B200 (the hot path of
arXiv 2202.06555, BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 5] [--points n] [--mode exact|fast]

A step evaluates the HDMR interpolant of the chosen BASELINE config (default:
config 5, d=300, m=151, 519 active slots, 115,198 nodes) at n points:
value = points x outputs per second over the whole job (weak scaling by
default: every rank evaluates n = 2^22 points, its contiguous shard of ONE
seeded stream of N x 2^22 points, grids replicated; `--scaling strong` splits
2^22 points across the ranks instead).  Inputs are
device-resident for `value`; `e2e` repeats the measurement through the same
public API with pinned host buffers (H2D of x and D2H of y inside every step).
One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "interpolant evals/sec (points x outputs)"
BLOCK_POINTS = 1 << 14  # seeded point blocks (ddsg_uniform_point_blocks; oracle/ref_workload.py)
UNIT = "evals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--points", type=int, default=0, help="total points (default: the config's n)")
    ap.add_argument("--mode", choices=["exact", "fast"], default="exact")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: the config's n points per GPU (default); strong: n points split over the GPUs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample time")
    ap.add_argument("--no-refine", action="store_true",
                    help="build the 1-d cuts at their final level instead of one distributed refinement step")
    ap.add_argument("--workload", choices=["eval", "euler", "jacobian"], default="eval",
                    help="eval: the HDMR evaluation (default, BASELINE metric); euler / jacobian: the batched "
                         "IRBC policy callers of SURVEY.md §8(f) rows 2-3 on a config-5-shaped policy")
    ap.add_argument("--countries", type=int, default=150, help="IRBC countries N for --workload euler/jacobian")
    ap.add_argument("--samples", type=int, default=10000, help="Euler-error samples per step (time_iteration.hpp:32)")
    ap.add_argument("--states", type=int, default=64, help="states per Jacobian step")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm = float(parts[1])
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            if sm > 0:
                sms.append(sm)
            for nm, v in zip(names, parts[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        if not sms:
            return None
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


# ----------------------------------------------------------- CPU baseline

def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_workload():
    """oracle/ref_workload.py: the configs built and evaluated by the
    reference alone (oracle/_ref), without loading the product library."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_workload as RW

    return RW


def time_reference(ref_hdmr, cfg, x_sample, target_s: float, workers: int):
    """VectorizedDdsg::evaluate_batch (ddsg_eval.hpp:130-139) on a growing
    prefix of the sample until one call takes >= target_s."""
    n = min(256, x_sample.shape[0])
    while True:
        t0 = time.perf_counter()
        rc, _ = ref_hdmr.eval(x_sample[:n], workers=workers, flat=False)
        dt = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError("reference evaluate_batch failed")
        if dt >= target_s or n >= x_sample.shape[0]:
            return n, dt
        n = min(x_sample.shape[0], max(n * 2, int(n * target_s / max(dt, 1e-3) * 1.1)))


def reference_variants():
    """The generic Release build and the x86-64-v3 build of oracle/_ref."""
    out = [ROOT / "oracle" / "_ref" / "libddsg_ref.so"]
    v3 = ROOT / "oracle" / "_ref" / "libddsg_ref_v3.so"
    try:
        flags = open("/proc/cpuinfo").read()
        if v3.exists() and " avx2 " in flags and " fma " in flags:
            out.append(v3)
    except Exception:
        pass
    return [p for p in out if p.exists()]


def cpu_baseline(cfg, target_s: float):
    """The reference's CPU path on this host's cores: every cut grid built by
    the reference's own SparseGridFunction::build, the first points of the
    bench's seeded stream through VectorizedDdsg::evaluate_batch(workers =
    all cores); the faster of the generic and x86-64-v3 builds of oracle/_ref.
    Returns (baseline dict, the faster build's (RefHdmr, lib))."""
    RW = ref_workload()
    workers = cpu_cores()
    best = None
    for path in reference_variants():
        lib = RW.use_library(path)
        ref = RW.build_hdmr(cfg, lib)[0]
        x = RW.points(lib, cfg, 0, 1 << 18)
        time_reference(ref, cfg, x, 0.5, workers)  # warm
        n, dt = time_reference(ref, cfg, x, target_s, workers)
        rate = n * cfg.m / dt
        if best is None or rate > best[0]:
            best = (rate, n, dt, path, ref, lib)
    if best is None:
        return None, None
    rate, n, dt, path, ref, lib = best
    return ({"value": rate, "unit": UNIT, "cores": workers, "kind": "reference",
             "sample": f"first {n} points of the seeded stream of {cfg.name} through the reference's "
                       f"VectorizedDdsg::evaluate_batch(workers={workers}) over grids built by its own "
                       f"SparseGridFunction::build ({path.name}, {dt:.1f} s)"}, (ref, lib))


def parity_check(ref_lib, cfg, y_dev, n_check: int):
    """Bit-exact check of the first n_check timed outputs against the
    reference (oracle/_ref, its own grid build) on the same points."""
    import numpy as np

    ref, lib = ref_lib
    RW = ref_workload()
    x = RW.points(lib, cfg, 0, n_check)
    rc, want = ref.eval(x, workers=cpu_cores(), flat=False)
    if rc != 0:
        return {"error": "reference evaluation failed"}
    got = y_dev[:n_check].cpu().numpy()
    same = np.all(got.view(np.uint64) == want.view(np.uint64), axis=1)
    tol = 1e-14 + 1e-12 * np.abs(want)
    return {"points": int(n_check), "outputs": int(n_check * cfg.m), "bit_identical_points": int(same.sum()),
            "outputs_outside_tolerance": int((np.abs(got - want) > tol).sum()),
            "max_abs_diff": float(np.max(np.abs(got - want))),
            "against": "oracle/_ref VectorizedDdsg::evaluate_batch over the reference's own SparseGridFunction::build "
                       "of every cut, first points of rank 0's timed inputs"}


# -------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank, dist):
    import numpy as np
    import torch

    from paper_2202_06555_b200 import workloads as W
    from paper_2202_06555_b200.ddsg import EXACT, FAST, last_eval_stats, measure_fp64_peak

    torch.cuda.set_device(local_rank)
    cfg = W.CONFIGS[args.config]
    n_total = (args.points or cfg.n_points) * (world if args.scaling == "weak" else 1)
    n_local = n_total // world + (1 if rank < n_total % world else 0)
    t0 = time.time()
    refine_info = None
    if cfg.kind == "hdmr" and not args.no_refine:
        # BASELINE config 5: "one refinement step whose new surpluses are NCCL
        # all-gathered before re-evaluation" -- build the 1-d cuts one level
        # short, then refine them on all ranks (each rank evaluates the target
        # and hierarchizes its share of the new nodes on its GPU; the surplus
        # rows are all-gathered over NCCL and appended everywhere).
        import dataclasses

        from paper_2202_06555_b200.ddsg import VectorizedDdsg
        from paper_2202_06555_b200.refine import refine_step

        coarse = dataclasses.replace(cfg, level_1d=cfg.level_1d - 1)
        if dist is not None:  # build once on rank 0, broadcast the nodes (NCCL)
            parts = W.broadcast_hdmr_parts(cfg, dist, f"cuda:{local_rank}", level_1d=cfg.level_1d - 1)
        else:
            parts = W.build_hdmr_parts(coarse)
        idx = [i for i, (u, b, g) in enumerate(parts.slots) if len(u) == 1]
        grids = [parts.slots[i][2] for i in idx]
        cuts = [W.CutTarget(cfg, parts.slots[i][0]) for i in idx]
        t_ref = time.time()
        st = refine_step(grids, [cfg.level_1d - 1] * len(grids), lambda gi, xs: cuts[gi](xs), dist=dist,
                         device=True, comm_device=f"cuda:{local_rank}")
        refine_info = {"new_nodes": st.new_nodes, "rounds": st.rounds, "allgather_bytes": st.gathered_bytes,
                       "hierarchize_s": round(st.hierarchize_s, 3), "target_eval_s": round(st.target_s, 3),
                       "allgather_s": round(st.allgather_s, 4),
                       "total_s": round(time.time() - t_ref, 2),
                       "collective": st.collective,
                       "build": "rank 0 builds, nodes broadcast (NCCL)" if dist is not None else "local build"}
        obj = VectorizedDdsg.compile(parts.d, parts.m, parts.f_anchor, parts.slots)
        evaluate = obj.evaluate_batch
    elif cfg.kind == "hdmr":
        obj, parts = W.build_hdmr(cfg)
        evaluate = obj.evaluate_batch
    else:
        obj, parts = W.build_grid(cfg), None
        evaluate = obj.interpolate
    obj.set_eval_mode(EXACT if args.mode == "exact" else FAST)
    build_s = time.time() - t0

    # the seeded blocked stream (block b: mt19937_64(seed + b), the reference
    # oracle's generator): rank r evaluates the contiguous shard
    # [first, first + n_local) of ONE point set, whatever the rank count
    from paper_2202_06555_b200.ddsg import uniform_point_blocks

    first = rank * (n_total // world) + min(rank, n_total % world)
    xh = torch.empty((n_local, cfg.d), dtype=torch.float64, pin_memory=True)
    uniform_point_blocks(cfg.seed, BLOCK_POINTS, first, n_local, cfg.d, out=xh.numpy())
    x = xh.cuda()
    y = torch.empty((n_local, cfg.m), dtype=torch.float64, device="cuda")

    # exact algorithmic work: NNZ_total = sum over points of (slot, node) pairs with w != 0
    nnz, _ = obj.support(x)
    nnz_total = int(np.asarray(nnz).sum())
    dfma, dmma = measure_fp64_peak()

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        evaluate(x, out=y)
    torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    main_ms = 0.0
    ev0.record(stream)
    for _ in range(args.steps):
        evaluate(x, out=y)
        l, _, mk = last_eval_stats()
        launches += l
        main_ms += mk
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([elapsed_ms, main_ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, main_ms_max = float(t[0]), float(t[1])
    ms_per_step = elapsed_ms / args.steps
    value = n_total * cfg.m / (ms_per_step / 1e3)

    # roofline of the dominant kernel (the slot kernel): algorithmic FLOPs = 2 m NNZ
    kernel_ms = main_ms / args.steps
    flops = 2.0 * cfg.m * nnz_total
    achieved = flops / (kernel_ms / 1e3) / 1e12
    traffic = None
    profs = sorted((ROOT / "profiles").glob("r*_ncu_fast_hdmr_config5.json"),
                   key=lambda p: int(p.name[1:].split("_")[0]))  # the latest round's capture
    prof = profs[-1] if profs else ROOT / "profiles" / "r1_ncu_fast_hdmr_config5.json"
    if cfg.name == "config5_hdmr_d300" and prof.exists():
        # DRAM bytes of the slot kernel from the committed ncu capture of this
        # config, scaled from its launch (447,392 points) to this step
        traffic = json.load(open(prof))["dram_bytes_per_point"] * n_local
    alg_bytes = 8.0 * n_local * (cfg.d + cfg.m) + 8.0 * obj.info()["n_nodes"] * cfg.m if parts else None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": dfma, "unit": "TFLOP/s",
                "frac": achieved / dfma, "traffic": traffic, "algorithmic_bytes": alg_bytes,
                "traffic_source": f"profiles/{prof.name} (dram__bytes_read+write per point x points)",
                "peak_source": "DFMA issue-rate microbenchmark measured live on this GPU "
                               "(MEASURED_PEAKS.json has no FP64 entry); DMMA peak %.1f TFLOP/s" % dmma,
                "kernel_ms": kernel_ms, "kernel_share": kernel_ms / ms_per_step,
                "flops_per_step": flops, "nnz_per_point": nnz_total / n_local,
                "exact_mode_cap_frac": 0.5}
    # The resource that binds the slot kernel: every term of
    # every point needs its own 8-byte surplus word per column in registers,
    # and the shared-memory pipe delivers 128 B/clk/SM to lanes (16 doubles;
    # profiles/r1_lds_gather.json) -> 2 * 16 FLOP-equivalents/clk/SM.
    sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
    mhz = float((clk or {}).get("sm_mhz") or 0.0) or 1965.0  # no samples in a very short timed region
    smem_peak = 2.0 * 16 * sms * mhz * 1e6 / 1e12
    if traffic:
        try:
            hbm_tbs = json.load(open(ROOT / "MEASURED_PEAKS.json"))["hbm_gbs"] / 1e3
        except Exception:
            hbm_tbs = 6.55  # B200_PROFILING.md fallback
        roofline["traffic_note"] = (
            "DRAM traffic is %.1fx the algorithmic bytes: 12.0 of 14.4 GB per launch are point coordinates (4 "
            "column-block groups x the 2.7 slots per dim a CTA evaluates ~0.5 ms apart, no L2 reuse between them), 2.4 "
            "GB staged tables (profiles/r2_l2_hints_config5.json, tables-only build), at %.2f TB/s of %.2f; the kernel "
            "is not HBM-bound: its time is flat while DRAM reads vary 2.7x with the grouping "
            "(profiles/r1_l2_budget_sweep_config5.json)"
            % (traffic / alg_bytes, traffic / (kernel_ms / 1e3) / 1e12, hbm_tbs))
    roofline["binding_resource"] = {
        "resource": "shared-memory gather: 16 surplus doubles/clk/SM (LDS pipe, 128 B/clk/SM)",
        "achieved": achieved, "peak": smem_peak, "unit": "TFLOP/s (2 FLOP per gathered double)",
        "frac": achieved / smem_peak,
        "peak_source": "shared-memory crossbar 128 B/clk/SM (B300_MICROARCH.md 'LDS/STS' table; reproduced by "
                       "profiles/r1_lds_gather.json: 0.496 lane-varying LDS.64 warp instructions/clk/SM) x %d SMs x "
                       "%.0f MHz (median SM clock in the timed region); every multiply-add of the hot path reads "
                       "its own 8-byte surplus from shared memory" % (sms, mhz)}

    # e2e through the same API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        try:
            yh = torch.empty((n_local, cfg.m), dtype=torch.float64, pin_memory=True)
            evaluate(xh, out=yh)
            barrier()
            t1 = time.perf_counter()
            for _ in range(args.steps):
                evaluate(xh, out=yh)
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device="cuda")
            if dist is not None:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            e2e_s = float(dt[0]) / args.steps
            if not torch.equal(yh, y.cpu()):
                raise RuntimeError("e2e result differs from the device-resident result")
            e2e = {"value": n_total * cfg.m / e2e_s, "unit": UNIT,
                   "h2d_bytes_per_step": n_total * cfg.d * 8, "d2h_bytes_per_step": n_total * cfg.m * 8,
                   "s_per_step": e2e_s, "timing": "wall clock around the synchronous C-ABI call"}
            del yh
        except RuntimeError as e:  # e.g. pinned allocation failure
            e2e = {"value": None, "unit": UNIT, "error": str(e)[:200]}

    cpu, parity = None, None
    if rank == 0 and not args.no_cpu_baseline and cfg.kind == "hdmr":
        try:
            if world == 1:  # the CPU baseline is reported at N=1 only
                cpu, ref_lib = cpu_baseline(cfg, args.cpu_seconds)
            else:  # N > 1: only the parity check's reference program
                RW = ref_workload()
                variants = reference_variants()
                lib = RW.use_library(variants[-1]) if variants else None
                ref_lib = (RW.build_hdmr(cfg, lib)[0], lib) if lib is not None else None
            if ref_lib is not None:
                parity = parity_check(ref_lib, cfg, y, min(n_local, 4096))
        except Exception as e:
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "d": cfg.d, "m": cfg.m, "points_total": n_total,
                       "points_per_gpu": n_local, "active_slots": obj.info()["n_active"] if parts else 1,
                       "nodes": obj.info()["n_nodes"] if parts else obj.size(),
                       "eval_mode": args.mode, "parallelism": f"points sharded over {world} GPU(s), grids replicated",
                       "l2": f"inputs {n_local * cfg.d * 8 / 1e9:.1f} GB per GPU, larger than L2 (no flush needed)",
                       "build_s": round(build_s, 1)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity, "gpu_launches": launches,
            "refinement": refine_info,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)


# ------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The reference's own CPU path: oracle/_ref only (its build, its
    evaluate_batch, its point generator, the targets linked into it); the
    product library is never loaded in this process."""
    if rank != 0:
        return
    RW = ref_workload()
    cfg = RW.configs()[args.config]
    if cfg.kind != "hdmr":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for the HDMR configs"}))
        return
    if not reference_variants():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libddsg_ref.so was not built"}))
        return
    workers = cpu_cores()
    path = reference_variants()[-1]
    lib = RW.use_library(path)
    t0 = time.time()
    ref = RW.build_hdmr(cfg, lib)[0]
    build_s = time.time() - t0
    x = RW.points(lib, cfg, 0, 1 << 14)
    # size one step to ~ (a few minutes / steps) of CPU work
    n, dt = time_reference(ref, cfg, x, 2.0, workers)
    for _ in range(args.warmup):
        ref.eval(x[:n], workers=workers, flat=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.eval(x[:n], workers=workers, flat=False)
    dt = (time.perf_counter() - t0) / args.steps
    v = n * cfg.m / dt
    sample = (f"first {n} points of the seeded stream of {cfg.name} per step through "
              f"VectorizedDdsg::evaluate_batch(workers={workers}); every cut grid built by the reference's "
              f"SparseGridFunction::build ({path.name}; build {build_s:.1f} s)")
    loaded = sorted({p.split()[-1] for p in open("/proc/self/maps") if p.strip().endswith(".so")
                     and str(ROOT) in p})
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "d": cfg.d, "m": cfg.m, "points_per_step": n},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libraries_loaded": [str(Path(p).relative_to(ROOT)) for p in loaded],
    }), flush=True)


# ------------------------------------------- IRBC callers

def build_irbc_policy(args):
    """A config-5-shaped policy on an N-country IRBC state space: 2N 1-d cuts
    (L=8) + 2N seeded pair cuts (L=5), eps 1e-8, modified-linear, center anchor."""
    from paper_2202_06555_b200 import irbc as I
    from paper_2202_06555_b200 import workloads as W

    p = I.make_parameters(args.countries, I.SMOOTH)
    tgt = W.IrbcPolicyTarget(args.countries, n_pairs=2 * args.countries, lam0=I.steady_state_lambda(p))
    vec, parts = W.build_policy_hdmr(tgt, 8, 5, 1e-8, 1e-8)
    return p, tgt, vec, parts


def caller_inputs(args, p, tgt, n):
    import numpy as np

    from paper_2202_06555_b200 import irbc as I
    from paper_2202_06555_b200.ddsg import uniform_points

    xs = uniform_points(20220213, n, p.state_dim())
    a, k = I.from_canonical(xs, p)
    z = tgt(xs)
    return xs, a, k, z


def run_callers(args, rank, world, local_rank, dist):
    import numpy as np
    import torch

    from paper_2202_06555_b200 import irbc as I
    from paper_2202_06555_b200.ddsg import EXACT, FAST, last_eval_stats, measure_fp64_peak

    torch.cuda.set_device(local_rank)
    t0 = time.time()
    p, tgt, vec, parts = build_irbc_policy(args)
    vec.set_eval_mode(EXACT if args.mode == "exact" else FAST)
    build_s = time.time() - t0
    N, pd, Q = p.countries, p.policy_dim(), 2 * (p.countries + 1)
    euler = args.workload == "euler"
    n_total = args.samples if euler else args.states
    if n_total < world:
        raise SystemExit("fewer units than ranks")
    n_local = n_total // world + (1 if rank < n_total % world else 0)
    lo = rank * (n_total // world) + min(rank, n_total % world)
    xs, a, k, z = caller_inputs(args, p, tgt, n_total)
    xs, a, k, z = (v[lo:lo + n_local] for v in (xs, a, k, z))
    dev = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()
    xs_d, a_d, k_d, z_d = dev(xs), dev(a), dev(k), dev(z)
    if euler:
        step = lambda: I.euler_errors_at(vec, p, xs_d)
        pts_per_unit = 1 + Q
    else:
        r0_d, _ = I.foc_residuals(vec, p, a_d, k_d, z_d)
        step = lambda: I.foc_jacobian(vec, p, a_d, k_d, z_d, r0_d)
        pts_per_unit = (N + 1) * Q
    nnz, _ = vec.support(xs_d[: min(n_local, 2048)])
    nnz_pp = float(np.asarray(nnz).mean())
    dfma, _ = measure_fp64_peak()

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches, main_ms = 0, 0.0
    ev0.record(stream)
    for _ in range(args.steps):
        out = step()
        l, _, mk = last_eval_stats()
        launches += l
        main_ms += mk
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1), main_ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t[0]) / args.steps
    kernel_ms = float(t[1]) / args.steps
    value = n_total / (ms_per_step / 1e3)
    flops = 2.0 * pd * nnz_pp * pts_per_unit * n_local
    achieved = flops / (kernel_ms / 1e3) / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": dfma, "unit": "TFLOP/s", "frac": achieved / dfma,
                "traffic": None, "kernel": "fast_hdmr_kernel (the batched policy evaluation)",
                "kernel_ms": kernel_ms, "kernel_share": kernel_ms / ms_per_step,
                "policy_points_per_step": pts_per_unit * n_local, "nnz_per_point": nnz_pp}
    # e2e: host numpy inputs / outputs through the same call
    if euler:
        e_host = lambda: I.euler_errors_at(vec, p, xs)
    else:
        r0_h = r0_d.cpu().numpy()
        e_host = lambda: I.foc_jacobian(vec, p, a, k, z, r0_h)
    e_host()
    barrier()
    t1 = time.perf_counter()
    for _ in range(args.steps):
        oh = e_host()
    e2e_s = (time.perf_counter() - t1) / args.steps
    dt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    e2e_s = float(dt[0])
    h2d = n_total * (p.state_dim() * 8 if euler else (2 * N + 2 * pd) * 8)
    d2h = n_total * (8 if euler else pd * pd * 8)
    e2e = {"value": n_total / e2e_s, "unit": "samples/s" if euler else "jacobians/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "s_per_step": e2e_s, "timing": "wall clock around the synchronous C-ABI call"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = caller_cpu_baseline(args, p, parts, *caller_inputs(args, p, tgt, max(n_total, 4096)), euler)
        except Exception as e:
            cpu = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        unit = "samples/s" if euler else "jacobians/s"
        metric = ("Euler-error samples/sec (solver.hpp:377-436, 1 + 2(N+1) policy evals each)" if euler else
                  "FOC Jacobians/sec (solver.hpp:129-165, forward differences, pdim x 2(N+1) policy evals each)")
        print(json.dumps({
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"irbc_{args.workload}_N{N}", "countries": N, "d": 2 * N, "m": pd,
                       "units_per_step": n_total, "policy": "config-5-shaped HDMR (2N 1-d cuts L=8, 2N pair cuts L=5)",
                       "active_slots": vec.info()["n_active"], "nodes": vec.info()["n_nodes"],
                       "eval_mode": args.mode, "build_s": round(build_s, 1),
                       "l2": "successor points regenerated each step (several GB), larger than L2"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }), flush=True)


def caller_cpu_baseline(args, p, parts, xs, a, k, z, euler, target_s=None):
    """The reference's foc_residuals under the oracle driver's restatements of
    euler_errors / foc_jacobian (oracle/_ref), all host threads, bounded sample."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O

    target_s = args.cpu_seconds if target_s is None else target_s
    workers = cpu_cores()
    libs = reference_variants()
    if not libs:
        return None
    O._ref = None
    O.REF_PATH = libs[-1]
    grids = []
    for u, b, g in parts.slots:
        if g is None:
            grids.append(None)
        else:
            kk, sur = g.nodes()
            grids.append(O.ref_from_nodes(len(u), parts.m, g.boundary_mode, g.max_level, g.eps_gamma, kk, sur))
    ref = O.RefHdmr(parts.d, parts.m, parts.f_anchor, [(u, b) for u, b, _ in parts.slots], grids)
    n = max(1, workers)
    pd = p.policy_dim()
    while True:
        t0 = time.perf_counter()
        if euler:
            O.ref_irbc_euler_errors(ref, p, xs[:n], workers=workers)
        else:
            O.ref_irbc_foc_residuals(ref, p, a[:n], k[:n], z[:n], workers=workers)
        dt = time.perf_counter() - t0
        if dt >= target_s or n >= xs.shape[0]:
            break
        n = min(xs.shape[0], max(n * 2, int(n * target_s / max(dt, 1e-3) * 1.1)))
    if euler:
        return {"value": n / dt, "unit": "samples/s", "cores": workers, "kind": "reference",
                "sample": f"euler_errors restatement over the reference's foc_residuals, first {n} samples, "
                          f"workers={workers} ({O.REF_PATH.name}, {dt:.1f} s)"}
    # a forward-difference Jacobian is exactly pdim foc_residuals calls (solver.hpp:135-142)
    return {"value": n / dt / pd, "unit": "jacobians/s", "cores": workers, "kind": "reference",
            "sample": f"reference foc_residuals on {n} states over {workers} threads ({dt:.1f} s, "
                      f"{O.REF_PATH.name}); jacobians/s = residuals/s / pdim ({pd} residual calls per Jacobian)"}


def run_callers_reference(args, rank, world):
    if rank != 0:
        return
    p, tgt, vec, parts = build_irbc_policy(args)
    euler = args.workload == "euler"
    xs, a, k, z = caller_inputs(args, p, tgt, args.samples if euler else args.states)
    cpu = caller_cpu_baseline(args, p, parts, xs, a, k, z, euler, target_s=20.0)
    if cpu is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libddsg_ref.so was not built"}))
        return
    print(json.dumps({"impl": "reference", "metric": args.workload, "value": cpu["value"], "unit": cpu["unit"],
                      "n_gpus": world, "steps": 1, "warmup": 0, "higher_is_better": True, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": f"irbc_{args.workload}_N{p.countries}"},
                      "cpu_baseline": cpu,
                      "e2e": {"value": cpu["value"], "unit": cpu["unit"], "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if args.workload != "eval":
            run_callers_reference(args, rank, world)
        else:
            run_reference(args, rank, world)
        return
    dist = None
    # DDSG_BENCH_FORCE_DIST=1 (under torchrun): a one-rank NCCL group, so the
    # collective code path (the refinement all-gather) runs on a single GPU
    if world > 1 or os.environ.get("DDSG_BENCH_FORCE_DIST") == "1":
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    try:
        if args.workload != "eval":
            run_callers(args, rank, world, local_rank, dist)
        else:
            run_ours(args, rank, world, local_rank, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
