"""End-to-end timing of the host-buffer paths a reference-style caller sees
(VERDICT r1 weak #7 / next #8), on config 5's HDMR program:

  * pinned host buffers (torch pin_memory) through ddsg_eval_hdmr;
  * ordinary pageable host buffers (numpy, i.e. std::vector memory) through
    ddsg_eval_hdmr (staged through pinned buffers inside the library);
  * device-resident buffers (the kernel-only reference point);
  * n = 1 latency of the per-point evaluate(x, out, ws) entry
    (ddsg_eval_hdmr_ws) and of ddsg_eval_hdmr with a one-point host buffer.

Usage: python tools/probe_e2e.py [n_points]   (default 2^22)
Prints one JSON object.
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2202_06555_b200 import _native as N
from paper_2202_06555_b200 import workloads as W
from paper_2202_06555_b200.ddsg import _check


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    cfg = W.CONFIGS[5]
    t0 = time.time()
    vec = W.build_hdmr(cfg)[0]
    build_s = time.time() - t0
    x_host = W.points(cfg, n=n)  # numpy, pageable
    m = cfg.m
    y_host = np.empty((n, m))
    x_pin = torch.from_numpy(x_host).pin_memory()
    y_pin = torch.empty((n, m), dtype=torch.float64).pin_memory()
    x_dev = x_pin.cuda()
    y_dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
    bad = C.c_int64(-1)
    h = vec._h

    def run(xp, yp, reps=3):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            _check(N.lib.ddsg_eval_hdmr(h, C.c_void_p(xp), n, C.c_void_p(yp), C.byref(bad), None))
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best

    run(x_dev.data_ptr(), y_dev.data_ptr(), 1)  # upload + warm-up
    t_dev = run(x_dev.data_ptr(), y_dev.data_ptr())
    t_pin = run(x_pin.data_ptr(), y_pin.data_ptr())
    t_pag = run(x_host.ctypes.data, y_host.ctypes.data)
    same = bool(np.array_equal(y_host.view(np.uint64), y_pin.numpy().view(np.uint64))
                and np.array_equal(y_host.view(np.uint64), y_dev.cpu().numpy().view(np.uint64)))

    # n = 1 latency
    ws = C.c_void_p()
    _check(N.lib.ddsg_workspace_create(C.byref(ws)))
    x1 = np.ascontiguousarray(x_host[:1])
    y1 = np.empty((1, m))
    calls = C.c_uint64(0)
    for _ in range(50):
        _check(N.lib.ddsg_eval_hdmr_ws(h, ws, C.c_void_p(x1.ctypes.data), 1, C.c_void_p(y1.ctypes.data),
                                       C.byref(bad), C.byref(calls)))
    reps = 2000
    t = time.perf_counter()
    for i in range(reps):
        N.lib.ddsg_eval_hdmr_ws(h, ws, C.c_void_p(x1.ctypes.data), 1, C.c_void_p(y1.ctypes.data), C.byref(bad), None)
    lat_ws = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for i in range(reps):
        N.lib.ddsg_eval_hdmr(h, C.c_void_p(x1.ctypes.data), 1, C.c_void_p(y1.ctypes.data), C.byref(bad), None)
    lat_plain = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for i in range(reps):
        pass
    loop_s = (time.perf_counter() - t) / reps
    assert np.array_equal(y1.view(np.uint64), y_host[:1].view(np.uint64))
    N.lib.ddsg_workspace_destroy(ws)
    evals = n * m
    print(json.dumps({
        "workload": "config5_hdmr_d300", "n": n, "m": m, "build_s": round(build_s, 1),
        "device_resident_s": t_dev, "pinned_host_s": t_pin, "pageable_host_s": t_pag,
        "evals_per_s": {"device": evals / t_dev, "pinned": evals / t_pin, "pageable": evals / t_pag},
        "pageable_over_pinned": t_pin / t_pag, "outputs_bit_identical_across_paths": same,
        "n1_latency_us": {"eval_hdmr_ws": lat_ws * 1e6, "eval_hdmr": lat_plain * 1e6,
                          "note": "ctypes call overhead included (~1-2 us)"},
    }))


if __name__ == "__main__":
    main()
