"""paper_2504_20655_b200 - B200-native batched Bellman-Ford warehouse routing.

A thin ctypes binding over libwr.so (include/wr.h). Argument marshalling
only: every step of the hot path runs in libwr's sm_100a kernels. PyTorch is
used for device memory, streams and torch.distributed plumbing. There is no
CPU fallback: importing this package without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np



_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WR_LIB") or os.path.join(_HERE, "libwr.so")   # WR_LIB: an experimental build

WR_OK, WR_EINVAL, WR_ENOMEM, WR_ENEGCYCLE, WR_EOVERFLOW, WR_EUNREACHABLE, WR_ETOOLARGE, WR_ECUDA, \
    WR_ENCCL, WR_EINTERNAL = range(10)
WR_I32, WR_F32 = 0, 1
WR_COO, WR_CSR = 0, 1
WR_BF_AUTO, WR_BF_FRONTIER, WR_BF_DENSE, WR_BF_NEARFAR = 0, 1, 2, 3
WR_ROUTE_ROWS32 = 1
WR_ROUTE_PAIRS = 2
WR_ROUTE_RANK_RESULTS = 4
WR_ROUTE_CLOSED = 8
WR_ROUTE_NEARFAR = 16
NCCL_UID_BYTES = 128
MAX_STOPS = 16
DEFAULT_CHUNK = 2903040
I32_INF = np.iinfo(np.int32).max

EXPORTS = [
    "wr_last_error", "wr_version", "wr_graph_load", "wr_graph_free", "wr_graph_info", "wr_bf_batch",
    "wr_route_cost", "wr_route_segmented", "wr_route_orders", "wr_segment_plan", "wr_route_count_reduction",
    "wr_orders_plan", "wr_plan_info", "wr_orders_local", "wr_orders_finish", "wr_plan_free", "wr_shard_range",
    "wr_release_cached", "wr_nccl_unique_id", "wr_ctx_create", "wr_ctx_free", "wr_ctx_info",
]


class WrError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libwr error {code}: {msg}")
        self.code = code


class GraphDesc(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int64), ("wtype", C.c_int32), ("format", C.c_int32),
                ("src", C.c_void_p), ("dst", C.c_void_p), ("row_ptr", C.c_void_p), ("col", C.c_void_p),
                ("w", C.c_void_p), ("xy", C.c_void_p), ("device", C.c_int32), ("z", C.c_void_p)]


class GraphInfo(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int64), ("wtype", C.c_int32), ("has_negative", C.c_int32),
                ("has_xy", C.c_int32), ("device", C.c_int32), ("device_bytes", C.c_int64),
                ("max_abs_weight", C.c_int32)]


class BfOpts(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("async_", C.c_int32), ("variant", C.c_int32),
                ("max_rounds", C.c_int32), ("hbm_budget", C.c_int64), ("ctx", C.c_void_p), ("shard", C.c_int32),
                ("reserved", C.c_int32)]


class BfStats(C.Structure):
    _fields_ = [("rounds_max", C.c_int32), ("relaxations", C.c_int64), ("segments", C.c_int32),
                ("tiles", C.c_int32), ("ms", C.c_float), ("negcycle_source", C.c_int32),
                ("kernel_launches", C.c_int64), ("visits", C.c_int64)]


class RouteOpts(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("async_", C.c_int32), ("m", C.c_int32), ("chunk", C.c_int64),
                ("hbm_budget", C.c_int64), ("pred_out", C.c_void_p), ("pred_rows", C.c_int64),
                ("flags", C.c_int32), ("depot", C.c_int32), ("ctx", C.c_void_p)]


class RouteStats(C.Structure):
    _fields_ = [("orders", C.c_int64), ("sources", C.c_int64), ("permutations", C.c_int64),
                ("stitch_candidates", C.c_int64), ("segments", C.c_int32), ("rounds_max", C.c_int32),
                ("relaxations", C.c_int64), ("ms", C.c_float), ("kernel_launches", C.c_int64),
                ("bf_ms", C.c_float), ("pred_ms", C.c_float), ("visits", C.c_int64),
                ("row_bits", C.c_int32), ("keyed", C.c_int32), ("tiles", C.c_int64), ("tile_sources", C.c_int32),
                ("reserved2", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("B", C.c_int64), ("S", C.c_int64), ("rank", C.c_int32), ("world", C.c_int32),
                ("src_lo", C.c_int64), ("src_hi", C.c_int64), ("order_lo", C.c_int64), ("order_hi", C.c_int64),
                ("send_count", C.c_int64), ("max_send", C.c_int64), ("wtype", C.c_int32)]


RESULT_DTYPE = np.dtype([("n", "<i4"), ("status", "<i4"), ("cost_bits", "<u4"), ("m_used", "<i4"),
                         ("rank", "<i8"), ("seq", "<i4", (MAX_STOPS,))])
assert RESULT_DTYPE.itemsize == 88


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                          "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    P = C.POINTER
    lib.wr_last_error.restype = C.c_char_p
    lib.wr_version.restype = i32
    lib.wr_graph_load.argtypes = [P(GraphDesc), P(vp)]
    lib.wr_graph_free.argtypes = [vp]
    lib.wr_graph_info.argtypes = [vp, P(GraphInfo)]
    lib.wr_bf_batch.argtypes = [vp, vp, i32, vp, i32, vp, vp, P(BfOpts), P(BfStats)]
    lib.wr_route_cost.argtypes = [i32, vp, i32, vp, i32, i64, vp, vp]
    lib.wr_route_segmented.argtypes = [vp, vp, i32, vp, i32, P(RouteOpts), vp]
    lib.wr_route_orders.argtypes = [vp, vp, vp, i64, vp, P(RouteOpts), vp, P(RouteStats)]
    lib.wr_segment_plan.argtypes = [vp, i32, i32, vp, i32]
    lib.wr_route_count_reduction.argtypes = [i32, vp, P(C.c_uint64), P(C.c_uint64)]
    lib.wr_orders_plan.argtypes = [vp, vp, vp, i64, vp, i32, i32, P(RouteOpts), P(vp)]
    lib.wr_nccl_unique_id.argtypes = [vp]
    lib.wr_ctx_create.argtypes = [i32, i32, vp, i32, P(vp)]
    lib.wr_ctx_free.argtypes = [vp]
    lib.wr_ctx_info.argtypes = [vp, P(i32), P(i32), P(i32)]
    lib.wr_plan_info.argtypes = [vp, P(PlanInfo)]
    lib.wr_orders_local.argtypes = [vp, vp, P(RouteOpts), P(RouteStats)]
    lib.wr_orders_finish.argtypes = [vp, vp, vp, P(RouteOpts), P(RouteStats)]
    lib.wr_plan_free.argtypes = [vp]
    lib.wr_shard_range.argtypes = [i64, i32, i32, P(i64), P(i64)]
    lib.wr_shard_range.restype = None
    lib.wr_release_cached.argtypes = [i32]
    for name in ["wr_release_cached", "wr_graph_load", "wr_graph_free", "wr_graph_info", "wr_bf_batch", "wr_route_cost",
                 "wr_route_segmented", "wr_route_orders", "wr_segment_plan", "wr_route_count_reduction",
                 "wr_orders_plan", "wr_plan_info", "wr_orders_local", "wr_orders_finish", "wr_plan_free",
                 "wr_nccl_unique_id", "wr_ctx_create", "wr_ctx_free", "wr_ctx_info"]:
        getattr(lib, name).restype = i32
    return lib


lib = _load()


def _check(rc):
    if rc != WR_OK:
        raise WrError(rc, lib.wr_last_error().decode(errors="replace"))


def _ptr(a):
    """Pointer of a numpy array or torch tensor (host or device), or None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def _arr(a, dtype):
    """numpy arrays are made contiguous with dtype; torch tensors pass through."""
    if a is None or not isinstance(a, np.ndarray) and hasattr(a, "data_ptr"):
        if a is not None:
            import torch
            tdt = {np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32,
                   np.uint32: torch.int32}[np.dtype(dtype).type]
            if a.dtype != tdt or not a.is_contiguous():
                raise TypeError(f"tensor must be contiguous {tdt}")
        return a
    return np.ascontiguousarray(a, dtype=dtype)


def _stream_ptr(stream):
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


def release_cached(device: int = 0):
    """Return libwr's idle pooled device memory to the driver."""
    _check(lib.wr_release_cached(device))


def shard_range(n: int, rank: int, world: int):
    lo, hi = C.c_int64(0), C.c_int64(0)
    lib.wr_shard_range(n, rank, world, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


class Graph:
    """a1: a warehouse graph resident on one device (wr_graph)."""

    def __init__(self, V, src=None, dst=None, w=None, xy=None, device=0, row_ptr=None, col=None, z=None):
        wdt = np.asarray(w).dtype if isinstance(w, np.ndarray) else None
        if wdt is None and hasattr(w, "dtype"):
            wdt = np.float32 if "float" in str(w.dtype) else np.int32
        wtype = WR_F32 if np.dtype(wdt) == np.float32 else WR_I32
        self._keep = []
        w = _arr(w, np.float32 if wtype == WR_F32 else np.int32)
        d = GraphDesc()
        d.V = int(V)
        d.wtype = wtype
        d.device = int(device)
        if row_ptr is not None:
            row_ptr = _arr(row_ptr, np.int64)
            col = _arr(col, np.int32)
            d.format = WR_CSR
            d.E = int(col.shape[0])
            d.row_ptr, d.col = _ptr(row_ptr), _ptr(col)
            self._keep += [row_ptr, col]
        else:
            src = _arr(src, np.int32)
            dst = _arr(dst, np.int32)
            d.format = WR_COO
            d.E = int(src.shape[0])
            d.src, d.dst = _ptr(src), _ptr(dst)
            self._keep += [src, dst]
        d.w = _ptr(w)
        if xy is not None:
            xy = _arr(xy, np.int32)
            d.xy = _ptr(xy)
            self._keep.append(xy)
        if z is not None:
            z = _arr(z, np.int32)
            d.z = _ptr(z)
            self._keep.append(z)
        self._keep.append(w)
        h = C.c_void_p()
        _check(lib.wr_graph_load(C.byref(d), C.byref(h)))
        self.handle = h
        self._keep = None
        self.V = int(V)
        self.wtype = wtype
        self.device = int(device)

    @classmethod
    def from_gen(cls, g, device=0, with_xy=True):
        return cls(g.V, g.src, g.dst, g.w, xy=g.xy if with_xy else None, device=device,
                   z=g.z if with_xy else None)

    def info(self) -> GraphInfo:
        i = GraphInfo()
        _check(lib.wr_graph_info(self.handle, C.byref(i)))
        return i

    def close(self):
        if getattr(self, "handle", None):
            lib.wr_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def vdtype(self):
        return np.float32 if self.wtype == WR_F32 else np.int32


def bf_batch(g: Graph, sources, targets=None, pred: bool = False, dist_out=None, pred_out=None,
             variant=WR_BF_AUTO, max_rounds=0, hbm_budget=0, stream=None, async_: bool = False,
             ctx: "Ctx" = None, shard: bool = False):
    """a3/a4: dist (S x T) and optional canonical pred (S x V).

    numpy in -> numpy out (host buffers); pass device tensors in dist_out /
    pred_out to keep results on the GPU. async_: with device outputs, return
    once the kernels are enqueued on `stream` (wr_bf_opts.async). ctx +
    shard: the sources are split over the context's ranks and every rank
    receives all rows. Returns (dist, pred, stats)."""
    src = _arr(sources, np.int32)
    S = int(src.shape[0])
    tg = _arr(targets, np.int32) if targets is not None else None
    T = int(tg.shape[0]) if tg is not None else g.V
    if dist_out is None:
        dist_out = np.empty((S, T), dtype=g.vdtype)
    if pred and pred_out is None:
        pred_out = np.empty((S, g.V), dtype=np.int32)
    o = BfOpts(_stream_ptr(stream), 1 if async_ else 0, variant, max_rounds, hbm_budget,
               ctx.handle if ctx is not None else None, 1 if shard else 0, 0)
    st = BfStats()
    _check(lib.wr_bf_batch(g.handle, _ptr(src), S, _ptr(tg), T if tg is not None else 0, _ptr(dist_out),
                           _ptr(pred_out) if pred else None, C.byref(o), C.byref(st)))
    return dist_out, (pred_out if pred else None), st


def route_cost(D, seqs, stream=None):
    """O4 on the device: left-to-right cost of each sequence (count x len)."""
    D = _arr(D, np.asarray(D).dtype if isinstance(D, np.ndarray) else np.int32)
    wtype = WR_F32 if D.dtype == np.float32 else WR_I32
    seqs = _arr(seqs, np.int32)
    if seqs.ndim == 1:
        seqs = seqs.reshape(1, -1)
    out = np.empty(seqs.shape[0], dtype=D.dtype)
    _check(lib.wr_route_cost(wtype, _ptr(D), int(D.shape[0]), _ptr(seqs), int(seqs.shape[1]), int(seqs.shape[0]),
                             _ptr(out), _stream_ptr(stream)))
    return out


def decode_cost(results, wtype):
    bits = np.asarray(results["cost_bits"], dtype=np.uint32)
    return bits.view(np.float32) if wtype == WR_F32 else bits.view(np.int32)


def route_segmented(g: Graph, stops, labels=None, m: int = 1, chunk: int = 0, stream=None, flags: int = 0):
    """a7: Theorem 3.1 route of one stop set (labels align with the sorted
    distinct stops; None -> O8 plan with K = m). flags=WR_ROUTE_PAIRS: the
    boundary-pair stitch (NEXT-1)."""
    stops = _arr(stops, np.int32)
    lab = _arr(labels, np.int32) if labels is not None else None
    out = np.zeros(1, dtype=RESULT_DTYPE)
    o = RouteOpts(_stream_ptr(stream), 0, m, chunk, 0, None, 0, flags)
    _check(lib.wr_route_segmented(g.handle, _ptr(stops), int(stops.shape[0]), _ptr(lab), m, C.byref(o),
                                  out.ctypes.data))
    return out[0]


def route_orders(g: Graph, order_ptr, order_nodes, m: int = 1, chunk: int = 0, results=None,
                 hbm_budget: int = 0, stream=None, pred_out=None, flags: int = 0, labels=None,
                 ctx: "Ctx" = None, depot: int = None):
    """a2..a9: route every order. Returns (results, stats); results is a
    RESULT_DTYPE numpy array unless a device buffer is passed. pred_out: an
    optional device int32 tensor (>= S rows x V) receiving the canonical
    predecessor rows (a4) of the distinct stops in ascending order (with a
    ctx: the rank's own block of sources, row 0 = its src_lo). labels: an
    optional segment label per order line (stitched routes over the
    caller's segments). ctx: shard over the context's ranks (collective).
    depot: route closed tours through this node (WR_ROUTE_CLOSED, NEXT-4)."""
    if depot is not None:
        flags |= WR_ROUTE_CLOSED
    ptr = _arr(order_ptr, np.int64)
    nodes = _arr(order_nodes, np.int32)
    lab = _arr(labels, np.int32) if labels is not None else None
    B = int(ptr.shape[0]) - 1
    if results is None:
        results = np.zeros(B, dtype=RESULT_DTYPE)
    o = RouteOpts(_stream_ptr(stream), 0, m, chunk, hbm_budget, _ptr(pred_out),
                  int(pred_out.shape[0]) if pred_out is not None else 0, flags,
                  int(depot) if depot is not None else 0, ctx.handle if ctx is not None else None)
    st = RouteStats()
    _check(lib.wr_route_orders(g.handle, _ptr(ptr), _ptr(nodes), B, _ptr(lab), C.byref(o), _ptr(results),
                               C.byref(st)))
    return results, st


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for wr_ctx_create (rank 0 makes it, the caller
    broadcasts it, e.g. torch.distributed.broadcast_object_list)."""
    buf = C.create_string_buffer(NCCL_UID_BYTES)
    _check(lib.wr_nccl_unique_id(buf))
    return buf.raw


class Ctx:
    """a9: libwr's multi-GPU context (wr_ctx): one per process and GPU,
    owning an NCCL communicator over `world` ranks."""

    def __init__(self, rank: int = 0, world: int = 1, uid: bytes = None, device: int = 0):
        h = C.c_void_p()
        ub = C.create_string_buffer(uid, NCCL_UID_BYTES) if uid is not None else None
        _check(lib.wr_ctx_create(rank, world, ub, device, C.byref(h)))
        self.handle = h
        self.rank, self.world, self.device = rank, world, device

    @classmethod
    def from_process_group(cls, device: int = None):
        """Bootstraps the communicator over torch.distributed (any backend):
        rank 0's unique id is broadcast to every rank."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        dev = torch.cuda.current_device() if device is None else device
        return cls(rank, world, obj[0], dev)

    def close(self):
        if getattr(self, "handle", None):
            lib.wr_ctx_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def segment_plan(xy, m: int, device: int = 0):
    xy = _arr(xy, np.int32).reshape(-1, 2)
    out = np.zeros(xy.shape[0], dtype=np.int32)
    _check(lib.wr_segment_plan(_ptr(xy), int(xy.shape[0]), m, _ptr(out), device))
    return out


def route_count_reduction(n_j):
    n_j = np.ascontiguousarray(n_j, dtype=np.int32)
    red, brute = C.c_uint64(0), C.c_uint64(0)
    _check(lib.wr_route_count_reduction(int(n_j.size), _ptr(n_j), C.byref(red), C.byref(brute)))
    return red.value, brute.value


class OrdersPlan:
    """a9 phases: plan (replicated) -> local BF + owned D entries -> all-gather
    (caller, torch.distributed) -> finish (route this rank's order block)."""

    def __init__(self, g: Graph, order_ptr, order_nodes, rank: int, world: int, m: int = 1, chunk: int = 0,
                 hbm_budget: int = 0, stream=None, pred_out=None, flags: int = 0, labels=None):
        self.g = g
        ptr = _arr(order_ptr, np.int64)
        nodes = _arr(order_nodes, np.int32)
        lab = _arr(labels, np.int32) if labels is not None else None
        self.opts = RouteOpts(_stream_ptr(stream), 0, m, chunk, hbm_budget, _ptr(pred_out),
                              int(pred_out.shape[0]) if pred_out is not None else 0, flags)
        h = C.c_void_p()
        _check(lib.wr_orders_plan(g.handle, _ptr(ptr), _ptr(nodes), int(ptr.shape[0]) - 1, _ptr(lab), rank, world,
                                  C.byref(self.opts), C.byref(h)))
        self.handle = h
        self.info = PlanInfo()
        _check(lib.wr_plan_info(h, C.byref(self.info)))

    def local(self, send):
        st = RouteStats()
        _check(lib.wr_orders_local(self.handle, _ptr(send), C.byref(self.opts), C.byref(st)))
        return st

    def finish(self, gathered, results=None):
        n = self.info.order_hi - self.info.order_lo
        if results is None:
            results = np.zeros(n, dtype=RESULT_DTYPE)
        st = RouteStats()
        _check(lib.wr_orders_finish(self.handle, _ptr(gathered), _ptr(results), C.byref(self.opts), C.byref(st)))
        return results, st

    def close(self):
        if getattr(self, "handle", None):
            lib.wr_plan_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
