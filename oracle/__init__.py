"""ctypes front-end of the CPU oracle (oracle/wr_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product path
(paper_2504_20655_b200) never imports this package, and this package never
imports the product path. Every function cites the reading it implements in
the C source header (O2..O8, P9 of DESIGN.md).

Parity unpinned: none of the functions below is unpinned; see DESIGN.md
"Oracle pins" for which test pins each one.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

I32, F32 = 0, 1
OK, EINVAL, ENOMEM, ENEGCYCLE, EOVERFLOW, EUNREACHABLE, ETOOLARGE = range(7)
I32_INF = np.iinfo(np.int32).max


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-pthread", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        vp, ip, lp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_longlong)
        L.orc_bf.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, C.c_int, vp, ip]
        L.orc_pred.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, C.c_int, vp, vp]
        L.orc_route_cost.argtypes = [C.c_int, vp, C.c_int, vp, C.c_int, vp]
        L.orc_exact_route.argtypes = [C.c_int, vp, C.c_int, vp, vp, lp]
        L.orc_exact_route_range.argtypes = [C.c_int, vp, C.c_int, C.c_longlong, C.c_longlong, vp, vp, lp]
        L.orc_exact_route_chunked.argtypes = [C.c_int, vp, C.c_int, C.c_longlong, vp, vp, lp, lp]
        L.orc_segmented_route.argtypes = [C.c_int, vp, C.c_int, vp, vp, vp, vp]
        L.orc_segmented_pairs_route.argtypes = [C.c_int, vp, C.c_int, vp, vp, vp, vp]
        L.orc_held_karp_route.argtypes = [C.c_int, vp, C.c_int, vp, vp, vp]
        L.orc_kmeans.argtypes = [vp, C.c_int, C.c_int, vp]
        L.orc_order_stops.argtypes = [vp, C.c_int, vp]
        L.orc_perm_rank.argtypes = [vp, C.c_int]
        L.orc_perm_rank.restype = C.c_longlong
        L.orc_route_count_reduction.argtypes = [C.c_int, vp, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]
        L.orc_bf_many.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, vp, C.c_int, vp, C.c_int]
        L.orc_pred_many.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int]
        L.orc_route_orders.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, vp, vp, C.c_longlong,
                                       C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, C.c_int, C.c_int]
        L.orc_closed_route_cost.argtypes = [C.c_int, vp, vp, vp, C.c_int, vp, C.c_int, vp]
        L.orc_exact_closed_route.argtypes = [C.c_int, vp, vp, vp, C.c_int, vp, vp, lp]
        L.orc_held_karp_closed_route.argtypes = [C.c_int, vp, vp, vp, C.c_int, vp, vp, lp]
        L.orc_segmented_closed_route.argtypes = [C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp]
        L.orc_segmented_pairs_closed_route.argtypes = [C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp]
        L.orc_certificate.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int]
        L.orc_certificate.restype = C.c_longlong
        L.orc_pred_certificate.argtypes = [C.c_int, C.c_longlong, vp, vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, lp]
        L.orc_pred_certificate.restype = C.c_longlong
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _wt(w):
    return I32 if np.asarray(w).dtype == np.int32 else F32


def _vdt(wt):
    return np.int32 if wt == I32 else np.float32


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: code {code}")
        self.code = code


def _graph(g):
    src = np.ascontiguousarray(g.src, dtype=np.int32)
    dst = np.ascontiguousarray(g.dst, dtype=np.int32)
    w = np.ascontiguousarray(g.w)
    if w.dtype not in (np.int32, np.float32):
        raise TypeError(w.dtype)
    if w.dtype == np.float32:
        w = np.where(w == 0, np.float32(0.0), w).astype(np.float32)  # -0.0 -> +0.0
    return g.V, src, dst, w


def bf(g, s: int):
    """O2: dist row from source s (int32 or float32 [V]); also rounds used."""
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    out = np.empty(V, dtype=_vdt(wt))
    rounds = C.c_int(0)
    rc = lib().orc_bf(V, src.size, _p(src), _p(dst), _p(w), wt, int(s), _p(out), C.byref(rounds))
    if rc:
        raise OracleError(rc, "bf")
    return out


def bf_rounds(g, s: int) -> int:
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    out = np.empty(V, dtype=_vdt(wt))
    rounds = C.c_int(0)
    rc = lib().orc_bf(V, src.size, _p(src), _p(dst), _p(w), wt, int(s), _p(out), C.byref(rounds))
    if rc:
        raise OracleError(rc, "bf")
    return rounds.value


def bf_many(g, sources, nthreads: int = None):
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    sources = np.ascontiguousarray(sources, dtype=np.int32)
    rows = np.empty((sources.size, V), dtype=_vdt(wt))
    rc = lib().orc_bf_many(V, src.size, _p(src), _p(dst), _p(w), wt, _p(sources), sources.size,
                           _p(rows), nthreads or os.cpu_count())
    if rc:
        raise OracleError(rc, "bf_many")
    return rows


def pred(g, s: int, dist):
    """O3: canonical predecessor row (-1 = none)."""
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    dist = np.ascontiguousarray(dist, dtype=_vdt(wt))
    out = np.empty(V, dtype=np.int32)
    rc = lib().orc_pred(V, src.size, _p(src), _p(dst), _p(w), wt, int(s), _p(dist), _p(out))
    if rc:
        raise OracleError(rc, "pred")
    return out


def pred_many(g, sources, dist, nthreads: int = None):
    """O3 for many rows (dist S x V from bf_many), on nthreads workers."""
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    sources = np.ascontiguousarray(sources, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=_vdt(wt))
    out = np.empty((sources.size, V), dtype=np.int32)
    rc = lib().orc_pred_many(V, src.size, _p(src), _p(dst), _p(w), wt, _p(sources), sources.size, _p(dist),
                             _p(out), nthreads or os.cpu_count())
    if rc:
        raise OracleError(rc, "pred_many")
    return out


def _D(D):
    D = np.ascontiguousarray(D)
    if D.dtype not in (np.int32, np.float32):
        raise TypeError(D.dtype)
    return D, _wt(D), D.shape[0]


def route_cost(D, seq):
    D, wt, n = _D(D)
    seq = np.ascontiguousarray(seq, dtype=np.int32)
    out = np.zeros(1, dtype=_vdt(wt))
    rc = lib().orc_route_cost(wt, _p(D), n, _p(seq), seq.size, _p(out))
    if rc:
        raise OracleError(rc, "route_cost")
    return out[0]


def exact_route(D):
    """O5: (cost, rank, seq) - first lexicographic minimum over n! sequences."""
    D, wt, n = _D(D)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    rank = C.c_longlong(0)
    rc = lib().orc_exact_route(wt, _p(D), n, _p(seq), _p(cost), C.byref(rank))
    if rc:
        raise OracleError(rc, "exact_route")
    return cost[0], rank.value, seq


def held_karp_route(D):
    """NEXT-2: exact route of up to 16 stops by the Held-Karp subset DP:
    (cost, rank, seq), the same result as exact_route."""
    D, wt, n = _D(D)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    rank = C.c_longlong(0)
    rc = lib().orc_held_karp_route(wt, _p(D), n, _p(seq), _p(cost), C.byref(rank))
    if rc:
        raise OracleError(rc, "held_karp_route")
    return cost[0], rank.value, seq


def exact_route_range(D, lo: int, hi: int):
    D, wt, n = _D(D)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    rank = C.c_longlong(0)
    rc = lib().orc_exact_route_range(wt, _p(D), n, lo, hi, _p(seq), _p(cost), C.byref(rank))
    if rc:
        raise OracleError(rc, "exact_route_range")
    return cost[0], rank.value, seq


def exact_route_chunked(D, chunk: int):
    D, wt, n = _D(D)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    rank, nch = C.c_longlong(0), C.c_longlong(0)
    rc = lib().orc_exact_route_chunked(wt, _p(D), n, chunk, _p(seq), _p(cost), C.byref(rank), C.byref(nch))
    if rc:
        raise OracleError(rc, "exact_route_chunked")
    return cost[0], rank.value, seq, nch.value


def segmented_route(D, labels):
    """O7: (cost, seq, (segment sequences evaluated, stitch candidates))."""
    D, wt, n = _D(D)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    counts = np.zeros(2, dtype=np.int64)
    rc = lib().orc_segmented_route(wt, _p(D), n, _p(labels), _p(seq), _p(cost), _p(counts))
    if rc:
        raise OracleError(rc, "segmented_route")
    return cost[0], seq, (int(counts[0]), int(counts[1]))


def segmented_pairs_route(D, labels):
    """NEXT-1 boundary-pair stitch: (cost, seq, (segment orders evaluated,
    stitch candidates))."""
    D, wt, n = _D(D)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    counts = np.zeros(2, dtype=np.int64)
    rc = lib().orc_segmented_pairs_route(wt, _p(D), n, _p(labels), _p(seq), _p(cost), _p(counts))
    if rc:
        raise OracleError(rc, "segmented_pairs_route")
    return cost[0], seq, (int(counts[0]), int(counts[1]))


def kmeans(xy, K: int):
    xy = np.ascontiguousarray(xy, dtype=np.int32).reshape(-1, 2)
    labels = np.zeros(xy.shape[0], dtype=np.int32)
    rc = lib().orc_kmeans(_p(xy), xy.shape[0], K, _p(labels))
    if rc:
        raise OracleError(rc, "kmeans")
    return labels


def order_stops(nodes):
    nodes = np.ascontiguousarray(nodes, dtype=np.int32)
    out = np.zeros(max(1, nodes.size), dtype=np.int32)
    n = lib().orc_order_stops(_p(nodes), nodes.size, _p(out))
    return out[:n].copy()


def perm_rank(seq) -> int:
    seq = np.ascontiguousarray(seq, dtype=np.int32)
    return lib().orc_perm_rank(_p(seq), seq.size)


def _legs(D, din, dout):
    D, wt, n = _D(D)
    din = np.ascontiguousarray(din, dtype=_vdt(wt)).reshape(n)
    dout = np.ascontiguousarray(dout, dtype=_vdt(wt)).reshape(n)
    return D, wt, n, din, dout


def closed_route_cost(D, din, dout, seq):
    """NEXT-4: cost of the closed tour depot -> seq -> depot (left to right)."""
    D, wt, n, din, dout = _legs(D, din, dout)
    seq = np.ascontiguousarray(seq, dtype=np.int32)
    out = np.zeros(1, dtype=_vdt(wt))
    rc = lib().orc_closed_route_cost(wt, _p(D), _p(din), _p(dout), n, _p(seq), seq.size, _p(out))
    if rc:
        raise OracleError(rc, "closed_route_cost")
    return out[0]


def _closed_call(fn, name, D, din, dout, *extra):
    D, wt, n, din, dout = _legs(D, din, dout)
    seq = np.zeros(n, dtype=np.int32)
    cost = np.zeros(1, dtype=_vdt(wt))
    tail = np.zeros(2, dtype=np.int64)
    args = [wt, _p(D), _p(din), _p(dout), n] + [_p(np.ascontiguousarray(e, dtype=np.int32)) for e in extra]
    rc = fn(*args, _p(seq), _p(cost), _p(tail) if extra else C.cast(C.c_void_p(tail.ctypes.data), C.POINTER(C.c_longlong)))
    if rc:
        raise OracleError(rc, name)
    return cost[0], seq, tail


def exact_closed_route(D, din, dout):
    """NEXT-4 exact closed tour over all n! orders: (cost, rank, seq)."""
    c, s, t = _closed_call(lib().orc_exact_closed_route, "exact_closed_route", D, din, dout)
    return c, int(t[0]), s


def held_karp_closed_route(D, din, dout):
    c, s, t = _closed_call(lib().orc_held_karp_closed_route, "held_karp_closed_route", D, din, dout)
    return c, int(t[0]), s


def segmented_closed_route(D, din, dout, labels):
    c, s, t = _closed_call(lib().orc_segmented_closed_route, "segmented_closed_route", D, din, dout, labels)
    return c, s, (int(t[0]), int(t[1]))


def segmented_pairs_closed_route(D, din, dout, labels):
    c, s, t = _closed_call(lib().orc_segmented_pairs_closed_route, "segmented_pairs_closed_route", D, din, dout,
                           labels)
    return c, s, (int(t[0]), int(t[1]))


def route_count_reduction(n_j):
    n_j = np.ascontiguousarray(n_j, dtype=np.int32)
    red, brute = C.c_ulonglong(0), C.c_ulonglong(0)
    lib().orc_route_count_reduction(n_j.size, _p(n_j), C.byref(red), C.byref(brute))
    return red.value, brute.value


def route_orders(g, orders, m: int = 1, nthreads: int = None, pairs: bool = False, depot: int = -1):
    """a2..a7 composed. Returns dict(n, seq [B,16] node ids, cost, rank, rc).
    depot >= 0: the NEXT-4 closed tour through that node (reading R4)."""
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    B = orders.B
    ptr = np.ascontiguousarray(orders.order_ptr, dtype=np.int64)
    nodes = np.ascontiguousarray(orders.order_nodes, dtype=np.int32)
    xy = np.ascontiguousarray(g.xy, dtype=np.int32)
    out_n = np.zeros(B, dtype=np.int32)
    out_seq = np.full((B, 16), -1, dtype=np.int32)
    out_cost = np.zeros(B, dtype=_vdt(wt))
    out_rank = np.zeros(B, dtype=np.int64)
    out_rc = np.zeros(B, dtype=np.int32)
    rc = lib().orc_route_orders(V, src.size, _p(src), _p(dst), _p(w), wt, _p(ptr), _p(nodes), B, m,
                                _p(xy), nthreads or os.cpu_count(), _p(out_n), _p(out_seq),
                                _p(out_cost), _p(out_rank), _p(out_rc), 1 if pairs else 0, int(depot))
    return dict(rc=rc, n=out_n, seq=out_seq, cost=out_cost, rank=out_rank, order_rc=out_rc)


def certificate(g, sources, dist, pred_rows=None, nthreads: int = None) -> int:
    """P9: number of rows failing the fixpoint certificate (0 = certified)."""
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    sources = np.ascontiguousarray(sources, dtype=np.int32)
    dist = np.ascontiguousarray(dist, dtype=_vdt(wt))
    pr = None if pred_rows is None else np.ascontiguousarray(pred_rows, dtype=np.int32)
    return lib().orc_certificate(V, src.size, _p(src), _p(dst), _p(w), wt, _p(sources), sources.size,
                                 _p(dist), _p(pr), nthreads or os.cpu_count())


def pred_certificate(g, sources, pred_rows, nthreads: int = None):
    """P9 from pred rows alone: (bad row count, first bad row or -1). A row
    passes iff pred is a tree rooted at its source whose path sums satisfy
    every arc (so they are the BF fixpoint) and pred is canonical (O3)."""
    V, src, dst, w = _graph(g)
    wt = _wt(w)
    sources = np.ascontiguousarray(sources, dtype=np.int32)
    pr = np.ascontiguousarray(pred_rows, dtype=np.int32)
    assert pr.shape == (sources.size, V)
    first = C.c_longlong(-1)
    bad = lib().orc_pred_certificate(V, src.size, _p(src), _p(dst), _p(w), wt, _p(sources), sources.size,
                                     _p(pr), nthreads or os.cpu_count(), C.byref(first))
    return bad, first.value
