"""Python mirror of the reference's interpolation API over the C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/ddsg/:
  SparseGridFunction.build / from_nodes / interpolate / nodes / quadrature
      (sparse_grid.hpp:84-179)
  VectorizedDdsg.compile (from DdsgFunction parts, hdmr.hpp:307-325 +
      ddsg_eval.hpp:40-74) / evaluate / evaluate_batch / quadrature
      (ddsg_eval.hpp:83-151)
Exceptions: InvalidArgument (std::invalid_argument), DomainError
(std::domain_error, with .task_id = lowest offending point like
task_error, runtime.hpp:71-92), BuildError (ddsg::build_error with .point).

Point arrays may be numpy arrays (host) or torch CUDA tensors (device
pointers, evaluated in place).  Evaluation always runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as N

ZERO_BOUNDARY = N.ZERO_BOUNDARY
MODIFIED_LINEAR = N.MODIFIED_LINEAR
EXACT = N.EVAL_EXACT
FAST = N.EVAL_FAST


class DdsgError(RuntimeError):
    pass


class InvalidArgument(DdsgError, ValueError):
    pass


class DomainError(DdsgError, ValueError):
    def __init__(self, msg: str, task_id: int = -1):
        super().__init__(msg)
        self.task_id = task_id


class BuildError(DdsgError):
    def __init__(self, msg: str, point: Sequence[float]):
        super().__init__(msg)
        self.point = list(point)


class OutOfMemory(DdsgError, MemoryError):
    pass


def _check(status: int, bad_index: int = -1) -> None:
    if status == N.OK:
        return
    msg = N.last_error()
    if status == N.INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == N.DOMAIN_ERROR:
        raise DomainError(msg, bad_index)
    if status == N.BUILD_ERROR:
        buf = (C.c_double * 64)()
        n = N.lib.ddsg_last_build_point(C.cast(buf, C.c_void_p), 64)
        raise BuildError(msg, [buf[i] for i in range(min(n, 64))])
    if status == N.OUT_OF_MEMORY:
        raise OutOfMemory(msg)
    raise DdsgError(f"status {status}: {msg}")


def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


def _as_points(x, dim: int):
    """Returns (array, n, is_single) with x as a C-contiguous float64 [n][dim]."""
    if isinstance(x, np.ndarray) or not hasattr(x, "data_ptr"):
        arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        single = arr.ndim == 1
        if single:
            arr = arr.reshape(1, -1)
        if arr.ndim != 2 or arr.shape[1] != dim:
            raise InvalidArgument("query dimension mismatch")
        return arr, arr.shape[0], single
    # torch tensor
    import torch

    if x.dtype != torch.float64:
        raise InvalidArgument("points must be float64")
    single = x.dim() == 1
    t = x.reshape(1, -1) if single else x
    if t.dim() != 2 or t.shape[1] != dim:
        raise InvalidArgument("query dimension mismatch")
    return t.contiguous(), t.shape[0], single


def _check_out(out, arr, n: int, m: int) -> None:
    """A caller-supplied output must be exactly what the C call writes:
    [n][m] float64, C-contiguous, in the same memory (host / device) as x."""
    if isinstance(out, np.ndarray):
        if not isinstance(arr, np.ndarray):
            raise InvalidArgument("out is host memory but the points are on the device")
        if out.dtype != np.float64 or out.shape != (n, m) or not out.flags["C_CONTIGUOUS"]:
            raise InvalidArgument(f"out must be a C-contiguous float64 array of shape ({n}, {m})")
        return
    if not hasattr(out, "data_ptr"):
        raise InvalidArgument("out must be a numpy array or a torch tensor")
    import torch

    if isinstance(arr, np.ndarray) or out.device != arr.device:
        raise InvalidArgument("out must be on the same device as the points")
    if out.dtype != torch.float64 or tuple(out.shape) != (n, m) or not out.is_contiguous():
        raise InvalidArgument(f"out must be a contiguous float64 tensor of shape ({n}, {m})")


class _DeviceScope:
    """For torch CUDA points: runs the C call on the tensor's device and, by
    default, on torch's current stream of that device (torch pool streams are
    non-blocking, so the legacy default stream would not order after them)."""

    def __init__(self, arr, stream):
        self.arr, self.stream, self.ctx = arr, stream, None

    def __enter__(self) -> int:
        if isinstance(self.arr, np.ndarray) or not getattr(self.arr, "is_cuda", False):
            return int(self.stream or 0)
        import torch

        self.ctx = torch.cuda.device(self.arr.device)
        self.ctx.__enter__()
        if self.stream is None:
            return int(torch.cuda.current_stream(self.arr.device).cuda_stream)
        return int(self.stream)

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)
        return False


def _alloc_out(like, n: int, m: int):
    if isinstance(like, np.ndarray):
        return np.empty((n, m), dtype=np.float64)
    import torch

    return torch.empty((n, m), dtype=torch.float64, device=like.device)


class _Evaluator:
    """Keeps a Python batch evaluator alive as a C callback."""

    def __init__(self, f: Callable[[np.ndarray], np.ndarray], dim: int, m: int):
        self.error: Optional[BaseException] = None

        def cb(xs, count, out, ctx):
            try:
                x = np.ctypeslib.as_array(xs, shape=(count, dim)).copy()
                y = np.asarray(f(x), dtype=np.float64).reshape(count, m)
                np.ctypeslib.as_array(out, shape=(count, m))[:] = y
                return 0
            except BaseException as e:  # surfaced after the C call returns
                self.error = e
                return 1

        self.c = N.BATCH_EVALUATOR(cb)


class SparseGridFunction:
    """Adaptive sparse grid (sparse_grid.hpp:72-351) backed by the GPU evaluator."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        dim, m, mode, lvl = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        eps, n = C.c_double(), C.c_int64()
        _check(N.lib.ddsg_grid_info(self._h, C.byref(dim), C.byref(m), C.byref(mode), C.byref(lvl),
                                    C.byref(eps), C.byref(n)))
        self.dim, self.out_dim, self.boundary_mode = dim.value, m.value, mode.value
        self.max_level, self.eps_gamma = lvl.value, eps.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N.lib is not None:
            N.lib.ddsg_grid_destroy(h)
            self._h = C.c_void_p(0)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # --- construction
    @staticmethod
    def build(f, dim: int, out_dim: int, max_level: int, eps_gamma: float = 0.0,
              mode: int = ZERO_BOUNDARY, norm: int = N.NORM_INF, ctx: int = 0) -> "SparseGridFunction":
        """f: Python callable xs[count][dim] -> out[count][out_dim], or the address
        of a C ddsg_batch_evaluator (int) with its ctx pointer."""
        out = C.c_void_p()
        if isinstance(f, int):
            st = N.lib.ddsg_grid_build(dim, out_dim, mode, max_level, eps_gamma, norm, C.c_void_p(f),
                                       C.c_void_p(ctx), C.byref(out))
            _check(st)
        else:
            ev = _Evaluator(f, dim, out_dim)
            st = N.lib.ddsg_grid_build(dim, out_dim, mode, max_level, eps_gamma, norm,
                                       C.cast(ev.c, C.c_void_p), None, C.byref(out))
            if ev.error is not None:
                raise ev.error
            _check(st)
        return SparseGridFunction(out.value)

    @staticmethod
    def from_nodes(dim: int, out_dim: int, max_level: int, eps_gamma: float, mode: int,
                   keys: np.ndarray, surplus: np.ndarray) -> "SparseGridFunction":
        keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(-1, dim) if dim > 0 else keys
        surplus = np.ascontiguousarray(surplus, dtype=np.float64).reshape(-1, out_dim) if out_dim > 0 else surplus
        if dim > 0 and out_dim > 0 and keys.shape[0] != surplus.shape[0]:
            raise InvalidArgument("sparse grid: node surplus length mismatch")
        out = C.c_void_p()
        n = keys.shape[0] if dim > 0 else 0
        _check(N.lib.ddsg_grid_create(dim, out_dim, mode, max_level, eps_gamma, n, _ptr(keys), _ptr(surplus),
                                      C.byref(out)))
        return SparseGridFunction(out.value)

    # --- accessors
    def size(self) -> int:
        n = C.c_int64()
        _check(N.lib.ddsg_grid_info(self._h, None, None, None, None, None, C.byref(n)))
        return n.value

    def nodes(self):
        """(keys [n][dim] uint32, surplus [n][m] float64) in stored order."""
        n = self.size()
        keys = np.empty((n, self.dim), dtype=np.uint32)
        sur = np.empty((n, self.out_dim), dtype=np.float64)
        _check(N.lib.ddsg_grid_nodes(self._h, _ptr(keys), _ptr(sur)))
        return keys, sur

    def quadrature(self) -> np.ndarray:
        q = np.empty(self.out_dim, dtype=np.float64)
        _check(N.lib.ddsg_grid_quadrature(self._h, _ptr(q)))
        return q

    def append(self, keys: np.ndarray, surplus: np.ndarray) -> None:
        """Appends refinement nodes; max_level follows the deepest level sum
        (the level of the reference build that admits it)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(-1, self.dim)
        surplus = np.ascontiguousarray(surplus, dtype=np.float64).reshape(-1, self.out_dim)
        if keys.shape[0] != surplus.shape[0]:
            raise InvalidArgument("grid append: keys and surplus row counts differ")
        _check(N.lib.ddsg_grid_append(self._h, keys.shape[0], _ptr(keys), _ptr(surplus)))
        lvl = C.c_int()
        _check(N.lib.ddsg_grid_info(self._h, None, None, None, C.byref(lvl), None, None))
        self.max_level = lvl.value

    def hierarchize(self, keys: np.ndarray, f_values: np.ndarray, device: bool = True) -> np.ndarray:
        """surplus = f - interpolate(grid, x(key)) for new nodes (sparse_grid.hpp:264-276);
        device=True evaluates on the GPU, False on the host (both bit-identical)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(-1, self.dim)
        if hasattr(f_values, "data_ptr") and getattr(f_values, "is_cuda", False):
            # device rows in, device rows out (ddsg_hierarchize with device buffers)
            import torch

            fv = f_values.reshape(-1, self.out_dim).contiguous().to(torch.float64)
            if fv.shape[0] != keys.shape[0]:
                raise InvalidArgument("hierarchize: f_values rows != keys rows")
            out = torch.empty_like(fv)
            with _DeviceScope(fv, None):
                _check(N.lib.ddsg_hierarchize(self._h, keys.shape[0], _ptr(keys), _ptr(fv), _ptr(out)))
            return out
        f_values = np.ascontiguousarray(f_values, dtype=np.float64).reshape(-1, self.out_dim)
        if f_values.shape[0] != keys.shape[0]:
            raise InvalidArgument("hierarchize: f_values rows != keys rows")
        out = np.empty_like(f_values)
        fn = N.lib.ddsg_hierarchize if device else N.lib.ddsg_hierarchize_host
        _check(fn(self._h, keys.shape[0], _ptr(keys), _ptr(f_values), _ptr(out)))
        return out

    def refine_candidates(self, level_sum: int) -> np.ndarray:
        """The batch the reference's build would insert after level sum s
        (sparse_grid.hpp:215-254), as heap keys [n][dim]."""
        n = C.c_int64()
        _check(N.lib.ddsg_grid_refine_candidates(self._h, level_sum, C.byref(n), None))
        keys = np.empty((n.value, self.dim), dtype=np.uint32)
        if n.value:
            _check(N.lib.ddsg_grid_refine_candidates(self._h, level_sum, C.byref(n), _ptr(keys)))
        return keys

    def set_eval_mode(self, mode: int) -> None:
        _check(N.lib.ddsg_grid_set_eval_mode(self._h, mode))

    # --- evaluation
    def interpolate(self, x, out=None, stream: Optional[int] = None):
        arr, n, single = _as_points(x, self.dim)
        if out is None:
            y = _alloc_out(arr, n, self.out_dim)
        else:
            _check_out(out, arr, n, self.out_dim)
            y = out
        bad = C.c_int64(-1)
        with _DeviceScope(arr, stream) as st_handle:
            st = N.lib.ddsg_eval_grid(self._h, _ptr(arr), n, _ptr(y), C.byref(bad), C.c_void_p(st_handle))
        _check(st, bad.value)
        return y[0] if single else y

    # --- JSON documents (serialize.hpp:31-77), through the C-ABI
    @staticmethod
    def from_json(text) -> "SparseGridFunction":
        """sparse_grid_from_json (serialize.hpp:54-77)."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        out = C.c_void_p()
        _check(N.lib.ddsg_grid_from_json(data, len(data), C.byref(out)))
        return SparseGridFunction(out.value)

    def to_json(self) -> str:
        """to_json(SparseGridFunction) (serialize.hpp:31-52) as save_json's text."""
        return _read_text(lambda buf, cap, n: N.lib.ddsg_grid_to_json(self._h, buf, cap, n))

    def support(self, x):
        arr, n, _ = _as_points(x, self.dim)
        nnz = np.empty(n, dtype=np.int64)
        h = np.empty(n, dtype=np.uint64)
        _check(N.lib.ddsg_grid_support(self._h, _ptr(arr), n, _ptr(nnz), _ptr(h), None))
        return nnz, h


class VectorizedDdsg:
    """VectorizedDdsg (ddsg_eval.hpp:28-165) over DdsgFunction parts.

    slots: list of (dims tuple, b, grid or None) in coeff_b order (empty index
    first, then (order, lexicographic)); grids are copied into the object."""

    def __init__(self, d: int, m: int, f_anchor, slots):
        self.d, self.out_dim = d, m
        self.slots = [(tuple(int(v) for v in dims), int(b), g) for dims, b, g in slots]
        fa = np.ascontiguousarray(f_anchor, dtype=np.float64)
        order = np.array([len(s[0]) for s in self.slots], dtype=np.int32)
        dims = np.array([v for s in self.slots for v in s[0]], dtype=np.int32)
        if dims.size == 0:
            dims = np.zeros(1, dtype=np.int32)
        b = np.array([s[1] for s in self.slots], dtype=np.int32)
        grids = (C.c_void_p * len(self.slots))(*[(s[2].handle.value if s[2] is not None else None) for s in self.slots])
        out = C.c_void_p()
        _check(N.lib.ddsg_hdmr_create(d, m, _ptr(fa), len(self.slots), _ptr(order), _ptr(dims), _ptr(b),
                                      C.cast(grids, C.c_void_p), C.byref(out)))
        self._h = out

    @staticmethod
    def compile(d: int, m: int, f_anchor, slots) -> "VectorizedDdsg":
        return VectorizedDdsg(d, m, f_anchor, slots)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N.lib is not None:
            N.lib.ddsg_hdmr_destroy(h)
            self._h = C.c_void_p(0)

    def info(self):
        d, m, ns, na, nn = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        _check(N.lib.ddsg_hdmr_info(self._h, C.byref(d), C.byref(m), C.byref(ns), C.byref(na), C.byref(nn)))
        return {"d": d.value, "m": m.value, "n_slots": ns.value, "n_active": na.value, "n_nodes": nn.value}

    def set_eval_mode(self, mode: int) -> None:
        _check(N.lib.ddsg_hdmr_set_eval_mode(self._h, mode))

    def evaluate_batch(self, xs, out=None, stream: Optional[int] = None):
        arr, n, single = _as_points(xs, self.d)
        if out is None:
            y = _alloc_out(arr, n, self.out_dim)
        else:
            _check_out(out, arr, n, self.out_dim)
            y = out
        bad = C.c_int64(-1)
        with _DeviceScope(arr, stream) as st_handle:
            st = N.lib.ddsg_eval_hdmr(self._h, _ptr(arr), n, _ptr(y), C.byref(bad), C.c_void_p(st_handle))
        _check(st, bad.value)
        return y[0] if single else y

    # --- JSON documents (serialize.hpp:84-145), through the C-ABI
    @staticmethod
    def from_json(text) -> "VectorizedDdsg":
        """ddsg_from_json (serialize.hpp:112-145) + compile.  .slots holds
        (dims, b, grid or None) in coeff_b order."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        out = C.c_void_p()
        _check(N.lib.ddsg_hdmr_from_json(data, len(data), C.byref(out)))
        self = VectorizedDdsg.__new__(VectorizedDdsg)
        self._h = out
        info = self.info()
        self.d, self.out_dim = info["d"], info["m"]
        self.slots = [self.slot(s) for s in range(info["n_slots"])]
        return self

    def slot(self, s: int):
        """Slot s (VectorizedDdsg::slots(), ddsg_eval.hpp:77): (dims, b, grid copy or None)."""
        order, b, g = C.c_int(), C.c_int32(), C.c_void_p()
        dims = np.zeros(max(self.d, 1), dtype=np.int32)
        _check(N.lib.ddsg_hdmr_slot(self._h, s, C.byref(order), _ptr(dims), C.byref(b), C.byref(g)))
        grid = SparseGridFunction(g.value) if g.value else None
        return tuple(int(v) for v in dims[: order.value]), int(b.value), grid

    def set_document(self, k_max: int, anchor_coords, rejected=(), cut_quadratures=None) -> None:
        """DdsgFunction fields a document carries beyond evaluation (k_max,
        anchor coords, rejected indices, cut quadratures [n_slots][m])."""
        coords = np.ascontiguousarray(anchor_coords, dtype=np.float64)
        if coords.shape != (self.d,):
            raise InvalidArgument("anchor coordinates length != dim")
        rej = [tuple(int(v) for v in u) for u in rejected]
        rorder = np.array([len(u) for u in rej] or [0], dtype=np.int32)
        rdims = np.array([v for u in rej for v in u] or [0], dtype=np.int32)
        q = None
        if cut_quadratures is not None:
            q = np.ascontiguousarray(cut_quadratures, dtype=np.float64)
            if q.shape != (len(self.slots), self.out_dim):
                raise InvalidArgument("cut quadratures must be [n_slots][m]")
        _check(N.lib.ddsg_hdmr_set_document(self._h, int(k_max), _ptr(coords), len(rej), _ptr(rorder), _ptr(rdims),
                                            _ptr(q)))

    def document(self):
        """(k_max, anchor coords, f_anchor, rejected list, cut quadratures or None)."""
        k, nr, nrd, hq = C.c_int(), C.c_int(), C.c_int64(), C.c_int()
        _check(N.lib.ddsg_hdmr_document(self._h, C.byref(k), None, None, C.byref(nr), C.byref(nrd), None, None,
                                        C.byref(hq), None))
        coords = np.empty(self.d)
        fa = np.empty(self.out_dim)
        rorder = np.zeros(max(nr.value, 1), dtype=np.int32)
        rdims = np.zeros(max(nrd.value, 1), dtype=np.int32)
        q = np.empty((len(self.slots), self.out_dim)) if hq.value else None
        _check(N.lib.ddsg_hdmr_document(self._h, None, _ptr(coords), _ptr(fa), None, None, _ptr(rorder), _ptr(rdims),
                                        None, _ptr(q)))
        rej, off = [], 0
        for r in range(nr.value):
            rej.append(tuple(int(v) for v in rdims[off: off + rorder[r]]))
            off += int(rorder[r])
        return k.value, coords, fa, rej, q

    def to_json(self) -> str:
        """to_json(DdsgFunction) (serialize.hpp:84-110) as save_json's text;
        needs set_document (or a document-loaded object)."""
        return _read_text(lambda buf, cap, n: N.lib.ddsg_hdmr_to_json(self._h, buf, cap, n))

    evaluate = evaluate_batch

    def support(self, x):
        arr, n, _ = _as_points(x, self.d)
        nnz = np.empty(n, dtype=np.int64)
        h = np.empty(n, dtype=np.uint64)
        _check(N.lib.ddsg_hdmr_support(self._h, _ptr(arr), n, _ptr(nnz), _ptr(h), None))
        return nnz, h

    def quadrature(self) -> np.ndarray:
        q = np.empty(self.out_dim, dtype=np.float64)
        _check(N.lib.ddsg_hdmr_quadrature(self._h, _ptr(q)))
        return q

    def uses_slot_kernel(self) -> bool:
        v = C.c_int()
        _check(N.lib.ddsg_hdmr_kernel_path(self._h, C.byref(v)))
        return bool(v.value)


def _read_text(writer) -> str:
    n = C.c_int64()
    _check(writer(None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(writer(C.cast(buf, C.c_void_p), n.value + 1, C.byref(n)))
    return buf.raw[: n.value].decode()


def last_eval_stats():
    """(kernel launches, device ms of the whole evaluation, device ms of the dominant kernel)."""
    launches, ms, main = C.c_int64(), C.c_double(), C.c_double()
    N.lib.ddsg_last_eval_stats(C.byref(launches), C.byref(ms), C.byref(main))
    return launches.value, ms.value, main.value


def measure_fp64_peak():
    """(DFMA TFLOP/s, DMMA TFLOP/s) measured on the current device."""
    a, b = C.c_double(), C.c_double()
    _check(N.lib.ddsg_measure_fp64_peak(C.byref(a), C.byref(b)))
    return a.value, b.value


def uniform_point_blocks(seed: int, block_points: int, first: int, n: int, dim: int, out=None) -> np.ndarray:
    """Points [first, first + n) of the blocked seeded stream: block b is
    std::mt19937_64(seed + b) + uniform_real_distribution(0,1), point-major
    (include/ddsg_b200.h).  out: optional C-contiguous float64 [n][dim] host
    array (e.g. a pinned torch tensor's numpy view)."""
    if out is None:
        out = np.empty((n, dim), dtype=np.float64)
    N.lib.ddsg_uniform_point_blocks(C.c_uint64(seed), block_points, first, n, dim, _ptr(out))
    return out


def uniform_points(seed: int, n: int, dim: int) -> np.ndarray:
    """std::mt19937_64 + uniform_real_distribution(0,1), point-major (oracles.hpp:45-53)."""
    out = np.empty((n, dim), dtype=np.float64)
    N.lib.ddsg_uniform_points(C.c_uint64(seed), n, dim, _ptr(out))
    return out
