"""CPU oracle for arXiv 1610.07394 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1610_07394_b200``) never imports it and shares no code
with it; see the header of ``oracle.c`` for the citations of every function.

This module is argument marshalling only: every computation happens in the
plain C of ``oracle.c`` (compiled with ``-O2 -ffp-contract=off``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-shared", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None

u64, i64, i32, f32, f64 = C.c_uint64, C.c_int64, C.c_int, C.c_float, C.c_double
P = C.c_void_p

_SIGS = {
    "or_simplex_volume": (u64, [i32, u64]),
    "or_simplex_contains": (i32, [i32, u64, P]),
    "or_enumerate_count": (u64, [i32, u64]),
    "or_stacked_volume": (u64, [i32, u64]),
    "or_bb_alpha": (f64, [i32, u64]),
    "or_vs2_recurrence": (u64, [u64]),
    "or_vs3_recurrence": (u64, [u64]),
    "or_vs3_arity3_recurrence": (u64, [u64]),
    "or_vsm_recurrence": (u64, [i32, u64, u64, u64]),
    "or_vsm_alpha": (f64, [i32, u64, u64, u64]),
    "or_floor_log2": (i32, [u64]),
    "or_lambda2": (i32, [u64, u64, P, P]),
    "or_rec2": (i32, [u64, u64, u64, P, P]),
    "or_lambda3": (i32, [u64, u64, u64, u64, P]),
    "or_rec3": (i32, [u64, u64, u64, u64, P]),
    "or_check_cover2_blocks": (i32, [u64, i32, P]),
    "or_check_cover3_blocks": (i32, [u64, i32, P]),
    "or_check_rec2": (i64, [u64]),
    "or_check_rec3": (i64, [u64]),
    "or_rank2_strict": (u64, [u64, u64]),
    "or_rank2_incl": (u64, [u64, u64]),
    "or_rank3": (u64, [u64, u64, u64]),
    "or_rank3_incl": (u64, [u64, u64, u64]),
    "or_domain_volume": (u64, [i32, i32, u64]),
    "or_thread_elem2": (i32, [i32, i32, u64, u64, u64, u64, u64, u64, P]),
    "or_thread_elem3": (i32, [i32, u64, u64, u64, u64, u64, u64, u64, u64, P]),
    "or_grid_blocks": (u64, [i32, i32, i32, u64, u64]),
    "or_padded_n": (u64, [u64]),
    "or_thread_dump": (i32, [i32, i32, i32, u64, u64, u64, u64, i32, P, u64]),
    "or_element_hits": (i32, [i32, i32, i32, u64, u64, u64, u64, i32, P, u64, P]),
    "or_column_work": (i64, [i32, i32, u64, u64, u64]),
    "or_index_write": (i32, [i32, i32, u64, P, i32]),
    "or_edm_dist": (f32, [P, u64, u64]),
    "or_edm": (i32, [u64, P, P]),
    "or_atm_term": (f32, [P, u64, u64, u64, f32]),
    "or_atm_sum": (f64, [u64, P, f32, u64, u64, i32]),
    "or_tc_pred": (i32, [P, u64, u64, u64, f32]),
    "or_tc_count": (u64, [u64, P, f32, u64, u64, i32]),
    "or_max_threads": (i32, []),
    "or_cs_array": (i32, [P, i32, u64, u64, P]),
    "or_cs_index": (i32, [i32, i32, u64, u64, u64, i32, P]),
    "or_cs_edm": (i32, [u64, P, u64, u64, i32, P]),
    "or_map_dump": (i32, [i32, i32, i32, u64, u64, u64, i32, P, u64]),
    "or_tile_layout2": (i32, [u64, u64, i32, i32, u64, u64, P, u64]),
    "or_cs_tiles2": (i32, [i32, u64, u64, i32, i32, u64, u64, P, i32, P]),
    "or_tile_layout3": (i32, [u64, u64, i32, u64, u64, P, u64]),
    "or_cs_tiles3": (i32, [u64, u64, i32, u64, u64, i32, P]),
    "or_below_segments": (i32, [u64, P, P]),
    "or_below_tiles": (u64, [i32, u64, P]),
    "or_below_element_hits": (i32, [i32, i32, u64, u64, P, u64, P]),
    "or_below_tile_layout": (i64, [i32, i32, u64, u64, P, u64]),
    "or_cs_below_tiles": (i32, [i32, i32, i32, u64, u64, P, i32, P]),
}


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        for name, (res, args) in _SIGS.items():
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = res, args
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _pts(points: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(points, dtype=np.float32)
    assert p.ndim == 2 and p.shape[1] == 3
    return p


# ---------------------------------------------------------------- geometry
def simplex_volume(m, n): return lib().or_simplex_volume(m, n)
def simplex_contains(m, n, x): return bool(lib().or_simplex_contains(m, n, _ptr(np.asarray(x, np.int64))))
def enumerate_count(m, n): return lib().or_enumerate_count(m, n)
def stacked_volume(m, n): return lib().or_stacked_volume(m, n)
def bb_alpha(m, n): return lib().or_bb_alpha(m, n)
def vs2(n): return lib().or_vs2_recurrence(n)
def vs3(n): return lib().or_vs3_recurrence(n)
def vs3_arity3(n): return lib().or_vs3_arity3_recurrence(n)
def vsm(m, n, beta=2, rden=2): return lib().or_vsm_recurrence(m, n, beta, rden)
def vsm_alpha(m, n, beta=2, rden=2): return lib().or_vsm_alpha(m, n, beta, rden)
def floor_log2(y): return lib().or_floor_log2(y)
def domain_volume(m, inclusive, n): return lib().or_domain_volume(m, int(inclusive), n)


# ---------------------------------------------------------------- maps
L3_INSIDE, L3_REFLECTED, L3_SPARE, L3_FILLER = 0, 1, 2, 3


def lambda2(wx, wy):
    x, y = C.c_uint64(), C.c_uint64()
    if lib().or_lambda2(wx, wy, C.byref(x), C.byref(y)):
        raise ValueError("lambda2 undefined for w_y = 0")
    return x.value, y.value


def rec2(wx, wy, N):
    x, y = C.c_uint64(), C.c_uint64()
    if lib().or_rec2(wx, wy, N, C.byref(x), C.byref(y)):
        raise ValueError("rec2 undefined")
    return x.value, y.value


def lambda3(N, wx, wy, wz):
    """Returns (class, (X,Y,Z), (I,J,K)); see or_lambda3."""
    o = np.zeros(6, np.int64)
    c = lib().or_lambda3(N, wx, wy, wz, _ptr(o))
    return c, tuple(int(v) for v in o[:3]), tuple(int(v) for v in o[3:])


def rec3(N, wx, wy, wz):
    o = np.zeros(3, np.int64)
    ok = lib().or_rec3(N, wx, wy, wz, _ptr(o))
    return tuple(int(v) for v in o) if ok else None


def check_cover2_blocks(N, corrupt=False):
    r = np.zeros(4, np.int64)
    assert lib().or_check_cover2_blocks(N, int(corrupt), _ptr(r)) == 0
    return dict(zip(["mapped", "missing", "duplicates", "outside"], r.tolist()))


def check_cover3_blocks(N, corrupt=False):
    r = np.zeros(10, np.int64)
    assert lib().or_check_cover3_blocks(N, int(corrupt), _ptr(r)) == 0
    keys = ["mapped", "missing", "duplicates", "outside", "inside", "reflected",
            "spare", "filler", "body_missing", "body_duplicates"]
    return dict(zip(keys, r.tolist()))


def check_rec2(N): return lib().or_check_rec2(N)
def check_rec3(N): return lib().or_check_rec3(N)


# ---------------------------------------------------------------- ranks / covers
def rank2_strict(i, j): return lib().or_rank2_strict(i, j)
def rank2_incl(i, j): return lib().or_rank2_incl(i, j)
def rank3(i, j, k): return lib().or_rank3(i, j, k)
def rank3_incl(i, j, k): return lib().or_rank3_incl(i, j, k)


def _mapc(bb) -> int:
    """Map code: True/"bb" -> 0 (bounding box), False/"lambda" -> 1, "enum" -> 2."""
    if isinstance(bb, str):
        return {"bb": 0, "lambda": 1, "enum": 2}[bb]
    return 0 if bb else 1


def thread_elem2(inclusive, bb, N, rho, wx, wy, tx, ty):
    e = np.zeros(3, np.int64)
    ok = lib().or_thread_elem2(int(inclusive), _mapc(bb), N, rho, wx, wy, tx, ty, _ptr(e))
    return (int(e[0]), int(e[1])) if ok else None


def thread_elem3(bb, N, rho, wx, wy, wz, a, b, c):
    e = np.zeros(3, np.int64)
    ok = lib().or_thread_elem3(_mapc(bb), N, rho, wx, wy, wz, a, b, c, _ptr(e))
    return (int(e[0]), int(e[1]), int(e[2])) if ok else None


def grid_blocks(m, inclusive, bb, N, G=1):
    return lib().or_grid_blocks(m, int(inclusive), _mapc(bb), N, G)


ORDERS = {"rows": 0, "squares": 1}


def padded_n(n) -> int:
    """n' = 2^ceil(log2 n), the grid size of "approach n from above"."""
    return lib().or_padded_n(n)


def thread_dump(m, inclusive, bb, n, rho, rank=0, G=1, order="rows") -> np.ndarray:
    N = padded_n(n) // rho
    length = grid_blocks(m, inclusive, bb, N, G) * rho ** m
    out = np.empty(length, np.uint64)
    assert lib().or_thread_dump(m, int(inclusive), _mapc(bb), n, rho, rank, G, ORDERS[order],
                                _ptr(out), length) == 0
    return out


def map_dump(m, inclusive, bb, N, rank=0, G=1, order="rows") -> np.ndarray:
    """Expected MAP_DUMP records (int32 x 4 per grid block, launch order)."""
    nb = grid_blocks(m, inclusive, bb, N, G)
    out = np.empty((nb, 4), np.int32)
    assert lib().or_map_dump(m, int(inclusive), _mapc(bb), N, rank, G, ORDERS[order], _ptr(out), nb) == 0
    return out


def tile_layout2(n, T, inclusive=False, bb=False, rank=0, G=1) -> np.ndarray:
    """pos_of_rank[p] for the lambda-order tile-blocked layout (or_tile_layout2)."""
    V = domain_volume(2, inclusive, n)
    out = np.empty(V, np.int64)
    assert lib().or_tile_layout2(n, T, int(inclusive), _mapc(bb), rank, G, _ptr(out), V) == 0
    return out


def to_tile_layout2(canonical: np.ndarray, n, T, inclusive=False, bb=False, rank=0, G=1) -> np.ndarray:
    """Permute a canonical packed array into shard `rank`'s tile-blocked array."""
    pos = tile_layout2(n, T, inclusive, bb, rank, G)
    own = pos >= 0
    out = np.empty(int(own.sum()), canonical.dtype)
    out[pos[own]] = canonical[own]
    return out


def cs_tiles2(payload, n, T, inclusive=False, bb=False, rank=0, G=1, points=None, nthreads=0):
    """Streaming checksum of 'index_write' / 'edm' in the tile-blocked layout."""
    cs = np.zeros(5, np.uint64)
    pp = _ptr(_pts(points)) if points is not None else None
    assert lib().or_cs_tiles2({"index_write": 0, "edm": 1}[payload], n, T, int(inclusive), _mapc(bb),
                              rank, G, pp, nthreads, _ptr(cs)) == 0
    return dict(zip(CS_KEYS, (int(v) for v in cs)))


def tile_layout3(n, T, bb=False, rank=0, G=1) -> np.ndarray:
    """pos_of_rank[p] for the m=3 tile-blocked layout (or_tile_layout3, reading E26); -1 = other shard."""
    V = domain_volume(3, False, n)
    out = np.empty(V, np.int64)
    assert lib().or_tile_layout3(n, T, _mapc(bb), rank, G, _ptr(out), V) == 0
    return out


def to_tile_layout3(canonical: np.ndarray, n, T, bb=False, rank=0, G=1) -> np.ndarray:
    """Permute a canonical packed triple array into shard `rank`'s tile-blocked array."""
    pos = tile_layout3(n, T, bb, rank, G)
    own = pos >= 0
    out = np.empty(int(own.sum()), canonical.dtype)
    out[pos[own]] = canonical[own]
    return out


def cs_tiles3(n, T, bb=False, rank=0, G=1, nthreads=0):
    """Streaming checksum of the m=3 index write in the tile-blocked layout."""
    cs = np.zeros(5, np.uint64)
    assert lib().or_cs_tiles3(n, T, _mapc(bb), rank, G, nthreads, _ptr(cs)) == 0
    return dict(zip(CS_KEYS, (int(v) for v in cs)))


def element_hits(m, inclusive, bb, n, rho, rank=0, G=1, hits=None, order="rows"):
    V = domain_volume(m, inclusive, n)
    if hits is None:
        hits = np.zeros(V, np.uint32)
    r = np.zeros(3, np.int64)
    assert lib().or_element_hits(m, int(inclusive), _mapc(bb), n, rho, rank, G, ORDERS[order],
                                 _ptr(hits), V, _ptr(r)) == 0
    return hits, dict(launched=int(r[0]), useful=int(r[1]), outside=int(r[2]))


def column_work(m, inclusive, n, rho, wx): return lib().or_column_work(m, int(inclusive), n, rho, wx)


# ---------------------------------------------------------------- payloads
def index_write(m, inclusive, n, elem_bytes=4) -> np.ndarray:
    V = domain_volume(m, inclusive, n)
    out = np.empty(V, np.uint32 if elem_bytes == 4 else np.uint64)
    lib().or_index_write(m, int(inclusive), n, _ptr(out), elem_bytes)
    return out


def edm(points) -> np.ndarray:
    p = _pts(points)
    n = p.shape[0]
    out = np.empty(n * (n - 1) // 2, np.float32)
    lib().or_edm(n, _ptr(p), _ptr(out))
    return out


def edm_dist(points, i, j): return lib().or_edm_dist(_ptr(_pts(points)), i, j)


def edm_dist_many(points, ii, jj) -> np.ndarray:
    p = _pts(points)
    f, pp = lib().or_edm_dist, _ptr(p)
    return np.array([f(pp, int(i), int(j)) for i, j in zip(ii, jj)], np.float32)


def atm_term(points, i, j, k, eps2): return lib().or_atm_term(_ptr(_pts(points)), i, j, k, eps2)


def atm_sum(points, eps2, k_lo=0, k_hi=None, nthreads=0):
    p = _pts(points)
    n = p.shape[0]
    return lib().or_atm_sum(n, _ptr(p), eps2, k_lo, n if k_hi is None else k_hi, nthreads)


def tc_pred(points, i, j, k, R): return bool(lib().or_tc_pred(_ptr(_pts(points)), i, j, k, R))


def tc_count(points, R, k_lo=0, k_hi=None, nthreads=0):
    p = _pts(points)
    n = p.shape[0]
    return lib().or_tc_count(n, _ptr(p), R, k_lo, n if k_hi is None else k_hi, nthreads)


def max_threads(): return lib().or_max_threads()


CS_KEYS = ("count", "s0", "s1", "mix", "xr")


def cs_array(arr: np.ndarray, p0=0):
    kind = {np.dtype(np.uint32): 0, np.dtype(np.uint64): 1, np.dtype(np.float32): 2}[arr.dtype]
    a = np.ascontiguousarray(arr)
    cs = np.zeros(5, np.uint64)
    lib().or_cs_array(_ptr(a), kind, p0, a.size, _ptr(cs))
    return dict(zip(CS_KEYS, (int(v) for v in cs)))


def cs_index(m, inclusive, n, lo=0, hi=None, nthreads=0):
    cs = np.zeros(5, np.uint64)
    lib().or_cs_index(m, int(inclusive), n, lo, n if hi is None else hi, nthreads, _ptr(cs))
    return dict(zip(CS_KEYS, (int(v) for v in cs)))


def cs_edm(points, lo=0, hi=None, nthreads=0):
    p = _pts(points)
    n = p.shape[0]
    cs = np.zeros(5, np.uint64)
    lib().or_cs_edm(n, _ptr(p), lo, n if hi is None else hi, nthreads, _ptr(cs))
    return dict(zip(CS_KEYS, (int(v) for v in cs)))


# ------------------------------------------------------------------ approach n from below (reading E28)
def below_segments(M):
    """(sizes, offsets) of the binary-digit segments of M tiles."""
    Ns, Os = np.zeros(64, np.uint64), np.zeros(64, np.uint64)
    p = lib().or_below_segments(M, _ptr(Ns), _ptr(Os))
    return [int(x) for x in Ns[:p]], [int(x) for x in Os[:p]]


def below_tiles(m, M) -> np.ndarray:
    """Tile records {x0, x1, x2, cls} of the below decomposition in launch order."""
    cnt = lib().or_below_tiles(m, M, None)
    out = np.zeros((cnt, 4), np.int32)
    lib().or_below_tiles(m, M, _ptr(out))
    return out


def below_element_hits(m, inclusive, n, T):
    """(hits per packed rank, {tiles, useful, outside}) of the below decomposition."""
    V = domain_volume(m, inclusive, n)
    hits = np.zeros(V, np.uint32)
    res = np.zeros(3, np.int64)
    assert lib().or_below_element_hits(m, int(inclusive), n, T, _ptr(hits), V, _ptr(res)) == 0
    return hits, dict(zip(("tiles", "useful", "outside"), (int(x) for x in res)))


def below_tile_layout(m, inclusive, n, T):
    """(pos_of_rank, layout length incl. holes) of the E29 tile-blocked layout."""
    V = domain_volume(m, inclusive, n)
    pos = np.zeros(V, np.int64)
    L = lib().or_below_tile_layout(m, int(inclusive), n, T, _ptr(pos), V)
    assert L >= 0
    return pos, int(L)


def cs_below_tiles(payload, m, inclusive, n, T, points=None, nthreads=0):
    """Streaming checksum of index write (payload "index_write") or EDM in the E29 layout."""
    cs = np.zeros(5, np.uint64)
    pts = _pts(points) if points is not None else np.zeros((1, 3), np.float32)
    assert lib().or_cs_below_tiles(1 if payload == "edm" else 0, m, int(inclusive), n, T, _ptr(pts), nthreads,
                                   _ptr(cs)) == 0
    return dict(zip(CS_KEYS, (int(v) for v in cs)))
