"""B200-native recursive simplex thread maps (arXiv 1610.07394) -- Python binding.

Thin ctypes marshalling over the C ABI of ``include/smap.h`` (``libsmap.so``,
built for sm_100a by ``_build.py``).  The functions here carry the C names;
every step of the hot path runs in the library's CUDA kernels.  PyTorch is
used only for device memory and streams.  There is no CPU fallback: importing
this package without the built library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsmap.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "smap.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                      " (no CPU fallback exists)")
_lib = C.CDLL(LIB_PATH)

# ------------------------------------------------------------------ enums
OK, E_INVALID, E_UNSUPPORTED, E_CUDA, E_NOMEM = range(5)
MAP = {"bb": 0, "lambda": 1, "enum": 2, "below": 3}
DIAG = {"strict": 0, "inclusive": 1}
GRAN = {"thread": 0, "tile": 1}
ORDER = {"rows": 0, "squares": 1}
LAYOUT = {"rows": 0, "tiles": 1}
PAYLOAD = {"index_write": 0, "edm": 1, "atm": 2, "tc": 3, "map_dump": 4, "hitcount": 5, "index_write_atm": 8,
           "thread_dump": 6, "empty": 7}
DEVICE_NONE = -2          # smap_plan(device=DEVICE_NONE): host-only plan (validation + closed forms)
RUN_CHECKSUM = 0x1
RUN_CHECKSUM_MIX = 0x2
RUN_XOR = 0x4
RUN_FAST_SQRT = 0x8      # EDM: sqrt.approx on the vector tile path (1e-5, not bit-exact)


class SmapError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"smap status {status}: {msg}")
        self.status = status


class PlanDesc(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int64), ("rho", C.c_int), ("map", C.c_int), ("diag", C.c_int),
                ("granularity", C.c_int), ("persistent", C.c_int), ("shard_rank", C.c_int),
                ("shard_count", C.c_int), ("device", C.c_int), ("order", C.c_int), ("layout", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("grid_blocks", C.c_uint64), ("launched_threads", C.c_uint64), ("useful_elems", C.c_uint64),
                ("wasted_threads", C.c_uint64), ("count", C.c_uint64), ("s0", C.c_uint64), ("s1", C.c_uint64),
                ("mix", C.c_uint64), ("sum", C.c_double), ("tc", C.c_uint64), ("xr", C.c_uint64),
                ("kernel_ms", C.c_float),
                ("launches", C.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = C.c_void_p
_SIGS = {
    "smap_plan": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(_P)]),
    "smap_plan_query": (C.c_int, [_P, C.POINTER(Stats)]),
    "smap_out_bytes": (C.c_int, [_P, C.c_int, C.POINTER(C.c_size_t)]),
    "smap_run": (C.c_int, [_P, C.c_int, _P, C.c_size_t, C.c_float, _P, C.c_size_t, C.c_uint32, _P]),
    "smap_run_host": (C.c_int, [_P, C.c_int, _P, C.c_size_t, C.c_float, _P, C.c_size_t, C.c_uint32, _P,
                                C.POINTER(Stats)]),
    "smap_stats_fetch": (C.c_int, [_P, C.POINTER(Stats)]),
    "smap_result_reduce": (C.c_int, [_P, _P, _P]),
    "smap_result_combine": (C.c_int, [_P, C.c_int, _P, _P]),
    "smap_volume": (C.c_uint64, [C.c_int, C.c_int64, C.c_int]),
    "smap_locate": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    "smap_destroy": (None, [_P]),
    "smap_last_error": (C.c_char_p, []),
    "smap_abi_version": (C.c_int, []),
    "smap_graph_capture": (C.c_int, [_P, C.c_int, _P, C.c_size_t, C.c_float, _P, C.c_size_t, C.c_uint32, _P,
                                     C.POINTER(_P)]),
    "smap_graph_launch": (C.c_int, [_P, _P]),
    "smap_graph_launches": (C.c_uint32, [_P]),
    "smap_graph_destroy": (None, [_P]),
    "smap_recursive_volume": (C.c_int, [C.c_int, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    "smap_recursive_volume_closed": (C.c_int, [C.c_int, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    "smap_alpha_limit": (C.c_double, [C.c_int, C.c_double, C.c_int]),
    "smap_r_star": (C.c_double, [C.c_int, C.c_int]),
    "smap_find_n0": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
    "smap_r_cover": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype, _fn.argtypes = _res, _args


def exported_symbols():
    """Names of every function declared in include/smap.h (for the ABI test)."""
    with open(HEADER_PATH) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(smap_[a-z_]+)\s*\(", src)) - {"smap_plan_s"})


def smap_last_error() -> str:
    return _lib.smap_last_error().decode()


def _check(status):
    if status != OK:
        raise SmapError(status, smap_last_error())


def smap_abi_version() -> int:
    return _lib.smap_abi_version()


def smap_volume(m: int, n: int, diag: str = "strict") -> int:
    return _lib.smap_volume(m, n, DIAG[diag])


class Plan:
    """Owns an smap_plan_t; see smap_plan.  `device` is the CUDA ordinal the
    plan lives on (resolved from the current device when planned with -1)."""

    def __init__(self, handle, desc: PlanDesc, device: int):
        self.handle = handle
        self.desc = desc
        self.device = device

    @property
    def m(self): return self.desc.m

    @property
    def n(self): return self.desc.n

    def __del__(self):
        # at interpreter shutdown the module globals may already be gone; the
        # process exit releases the device memory then
        try:
            smap_destroy(self)
        except (TypeError, AttributeError):
            pass


def smap_plan(m: int, n: int, rho: int, map: str = "lambda", diag: str = "strict", granularity: str = "thread",
              persistent: int = 0, shard_rank: int = 0, shard_count: int = 1, device: int = -1,
              order: str = "rows", layout: str = "rows") -> Plan:
    d = PlanDesc(m, n, rho, MAP[map], DIAG[diag], GRAN[granularity], persistent, shard_rank, shard_count, device,
                 ORDER[order], LAYOUT[layout])
    h = _P()
    _check(_lib.smap_plan(C.byref(d), C.byref(h)))
    dev = device
    if device == -1:
        import torch
        dev = torch.cuda.current_device()
    return Plan(h, d, dev)


def smap_destroy(plan: Plan):
    if plan is not None and getattr(plan, "handle", None):
        _lib.smap_destroy(plan.handle)
        plan.handle = None


def smap_plan_query(plan: Plan) -> dict:
    st = Stats()
    _check(_lib.smap_plan_query(plan.handle, C.byref(st)))
    return st.as_dict()


def smap_locate(plan: Plan, *elem) -> tuple:
    """(shard, position) of element (i, j[, k]) in the plan's output layout (host, O(1))."""
    e = (C.c_int64 * 3)(*(list(elem) + [0] * (3 - len(elem))))
    sh, pos = C.c_int(), C.c_uint64()
    _check(_lib.smap_locate(plan.handle, e, C.byref(sh), C.byref(pos)))
    return sh.value, pos.value


def smap_out_bytes(plan: Plan, payload: str) -> int:
    b = C.c_size_t()
    _check(_lib.smap_out_bytes(plan.handle, PAYLOAD[payload], C.byref(b)))
    return b.value


def _ptr(x):
    """Address of a ctypes-compatible buffer: an int (raw pointer), a torch
    tensor or a numpy array, or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):                       # numpy (host) array
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _nbytes(x):
    if x is None:
        return 0
    if hasattr(x, "untyped_storage"):
        return x.numel() * x.element_size()
    return x.nbytes


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return stream if isinstance(stream, int) else stream.cuda_stream


def _device_buffer(plan: Plan, x, what: str, nbytes=None, fp32_points=False):
    """(pointer, bytes) of a DEVICE buffer for smap_run: a contiguous torch CUDA
    tensor on the plan's device, or a raw device pointer (int) with an explicit
    byte count.  Host arrays are refused (use smap_run_host)."""
    if x is None:
        return None, 0
    if isinstance(x, int):
        if nbytes is None:
            raise ValueError(f"{what}: a raw pointer needs an explicit {what}_bytes")
        return x, int(nbytes)
    if not hasattr(x, "is_cuda"):
        raise TypeError(f"{what} must be a CUDA tensor (or a raw device pointer); host arrays go through smap_run_host")
    if not x.is_cuda:
        raise ValueError(f"{what} is a host tensor; smap_run takes device buffers (use smap_run_host for host points)")
    if x.device.index != plan.device:
        raise ValueError(f"{what} is on cuda:{x.device.index}, the plan on cuda:{plan.device}")
    if not x.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if fp32_points:
        import torch
        if x.dtype != torch.float32 or x.numel() < 3 * plan.n:
            raise ValueError(f"{what} must be float32 with at least n x 3 = {3 * plan.n} elements "
                             f"(got {x.dtype}, {x.numel()})")
    return x.data_ptr(), _nbytes(x) if nbytes is None else int(nbytes)


def _record_ptr(x, what: str, count: int = 1):
    """Pointer of a DEVICE result-record buffer of `count` 56-byte records: a
    contiguous CUDA tensor of at least 56 * count bytes, or a raw device
    pointer (the caller vouches for its size).  Host arrays are refused."""
    if x is None or isinstance(x, int):
        return x
    if not getattr(x, "is_cuda", False):
        raise TypeError(f"{what} must be a CUDA tensor (7 int64 per record) or a raw device pointer")
    if not x.is_contiguous() or _nbytes(x) < 56 * count:
        raise ValueError(f"{what} must be contiguous with at least {56 * count} bytes (got {_nbytes(x)})")
    return x.data_ptr()


def smap_run(plan: Plan, payload: str, points=None, param: float = 0.0, out=None, flags: int = 0,
             stream=None, points_bytes=None, out_bytes=None):
    """Asynchronous launch on `stream` (default: torch's current stream).
    points / out: contiguous CUDA tensors on the plan's device (points float32,
    n x 3), or raw device pointers with explicit points_bytes / out_bytes."""
    pp, pb = _device_buffer(plan, points, "points", points_bytes, fp32_points=True)
    op, ob = _device_buffer(plan, out, "out", out_bytes)
    _check(_lib.smap_run(plan.handle, PAYLOAD[payload], pp, pb, float(param), op, ob, flags, _stream(stream)))


def smap_run_host(plan: Plan, payload: str, host_points=None, param: float = 0.0, out=None, flags: int = 0,
                  stream=None, out_bytes=None) -> dict:
    """End-to-end call with a HOST point array (float32 n x 3, numpy or a CPU
    tensor, pinned recommended; copied H2D inside), results copied back to
    host; synchronous.  `out` stays a device tensor: the packed outputs are
    consumed on the device, only the 56-byte result record comes back."""
    hp, hb = None, 0
    if host_points is not None:
        if getattr(host_points, "is_cuda", False):
            raise ValueError("host_points is a CUDA tensor; use smap_run for device points")
        import numpy as np
        a = host_points.numpy() if hasattr(host_points, "numpy") else host_points
        if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous or a.size < 3 * plan.n:
            raise ValueError("host_points must be a contiguous float32 array with at least n x 3 elements")
        hp, hb = _ptr(host_points), a.nbytes
    op, ob = _device_buffer(plan, out, "out", out_bytes)
    st = Stats()
    _check(_lib.smap_run_host(plan.handle, PAYLOAD[payload], hp, hb, float(param), op, ob, flags, _stream(stream),
                              C.byref(st)))
    return st.as_dict()


class Graph:
    """Owns an smap_graph_t (one captured step of a plan); keeps the plan and
    the bound buffers alive for as long as the graph exists."""

    def __init__(self, handle, plan, keep):
        self.handle = handle
        self.plan = plan
        self._keep = keep

    @property
    def launches(self) -> int:
        return _lib.smap_graph_launches(self.handle)

    def __del__(self):
        try:
            if self.handle:
                _lib.smap_graph_destroy(self.handle)
                self.handle = None
        except (TypeError, AttributeError):
            pass


def smap_graph_capture(plan: Plan, payload: str, points=None, param: float = 0.0, out=None, flags: int = 0,
                       record=None, points_bytes=None, out_bytes=None) -> Graph:
    """Capture one step (smap_run + smap_result_reduce into `record`, a device
    tensor of 7 int64) into a CUDA graph; replay it with smap_graph_launch."""
    pp, pb = _device_buffer(plan, points, "points", points_bytes, fp32_points=True)
    op, ob = _device_buffer(plan, out, "out", out_bytes)
    if record is not None and not isinstance(record, int):
        _device_buffer(plan, record, "record")                # on the plan's device, contiguous
    rp = _record_ptr(record, "record")
    h = _P()
    _check(_lib.smap_graph_capture(plan.handle, PAYLOAD[payload], pp, pb, float(param), op, ob, flags, rp,
                                   C.byref(h)))
    return Graph(h, plan, (points, out, record))


def smap_graph_launch(graph: Graph, stream=None):
    _check(_lib.smap_graph_launch(graph.handle, _stream(stream)))


def smap_stats_fetch(plan: Plan) -> dict:
    st = Stats()
    _check(_lib.smap_stats_fetch(plan.handle, C.byref(st)))
    return st.as_dict()


RESULT_FIELDS = ("count", "s0", "s1", "mix", "tc", "xr", "sum")


def smap_result_reduce(plan: Plan, dst, stream=None):
    """Asynchronously reduce the last run's results into `dst`, a DEVICE tensor
    of 7 int64 (count, s0, s1, mix, tc, xr, bits of the fp64 sum) -- ready for
    an all-reduce of dst[:5] (exact mod 2^64), an xor of dst[5] and a sum of
    dst[6:].view(float64)."""
    _check(_lib.smap_result_reduce(plan.handle, _record_ptr(dst, "dst"), _stream(stream)))


def smap_result_combine(records, count: int, dst, stream=None):
    """Asynchronously combine `count` device records (7 int64 each, contiguous)
    into `dst` (7 int64 on the device): the cross-rank step after an
    all-gather of every rank's smap_result_reduce output, in one kernel."""
    _check(_lib.smap_result_combine(_record_ptr(records, "records", max(int(count), 1)), int(count),
                                    _record_ptr(dst, "dst"), _stream(stream)))


def result_dict(rec) -> dict:
    """Host view of a 6 x int64 result record."""
    import numpy as np
    a = rec.cpu().numpy() if hasattr(rec, "cpu") else np.asarray(rec)
    u = a.view(np.uint64)
    d = dict(zip(RESULT_FIELDS[:6], (int(x) for x in u[:6])))
    d["sum"] = float(a[6:7].view(np.float64)[0])
    return d


# ------------------------------------------------------------------ volume analysis (host only, NEXT-4)
def smap_recursive_volume(m: int, n: int, beta: int = 2, r_den: int = 2, closed: bool = False) -> int:
    """V(S_n^m) of the recursive orthotope set with r = 1/r_den and arity beta
    (recurrence, or the closed form of Eq. generic-m with closed=True)."""
    v = C.c_uint64()
    fn = _lib.smap_recursive_volume_closed if closed else _lib.smap_recursive_volume
    _check(fn(m, n, beta, r_den, C.byref(v)))
    return v.value


def smap_alpha_limit(m: int, r: float = 0.5, beta: int = 2) -> float:
    return _lib.smap_alpha_limit(m, r, beta)


def smap_r_star(m: int, beta: int = 2) -> float:
    return _lib.smap_r_star(m, beta)


def smap_find_n0(m: int, r: float, beta: int, n_max: int) -> tuple:
    """(n0 or None, V(S)/V(Delta_{n-1}) at n_max)."""
    n0, ratio = C.c_uint64(), C.c_double()
    _check(_lib.smap_find_n0(m, r, beta, n_max, C.byref(n0), C.byref(ratio)))
    return (n0.value or None), ratio.value


def smap_r_cover(m: int, beta: int, n0: int, n_max: int) -> float:
    r = C.c_double()
    _check(_lib.smap_r_cover(m, beta, n0, n_max, C.byref(r)))
    return r.value


# ------------------------------------------------------------------ torch conveniences
def out_dtype(plan: Plan, payload: str):
    import torch
    if payload == "edm":
        return torch.float32
    if payload in ("index_write", "index_write_atm"):
        return torch.int64 if smap_volume(plan.m, plan.n, "inclusive" if plan.desc.diag else "strict") > (1 << 32) \
            else torch.int32
    if payload == "hitcount":
        return torch.int32
    if payload == "map_dump":
        return torch.int32
    if payload == "thread_dump":
        return torch.int64
    return None


def alloc_out(plan: Plan, payload: str, device="cuda", zero: bool = False):
    """Device tensor sized by smap_out_bytes (int32/int64 views of uint32/uint64 data)."""
    import torch
    nb = smap_out_bytes(plan, payload)
    if nb == 0:
        return None
    dt = out_dtype(plan, payload)
    cnt = nb // torch.empty((), dtype=dt).element_size()
    return (torch.zeros if zero else torch.empty)(cnt, dtype=dt, device=device)


__all__ = ["smap_plan", "smap_plan_query", "smap_out_bytes", "smap_run", "smap_run_host", "smap_stats_fetch",
           "smap_result_reduce", "smap_result_combine", "smap_graph_capture", "smap_graph_launch", "Graph",
           "smap_volume", "smap_destroy", "smap_last_error", "smap_abi_version", "Plan", "SmapError",
           "alloc_out", "exported_symbols", "RUN_CHECKSUM", "RUN_CHECKSUM_MIX", "RUN_XOR",
           "RUN_FAST_SQRT"]
