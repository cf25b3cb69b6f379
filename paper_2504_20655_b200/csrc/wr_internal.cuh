// wr_internal.cuh - shared internals of libwr (not part of the ABI).
// Everything here is the CUDA path; it shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>
#include <string>
#include <vector>

#include "../../include/wr.h"

namespace wr {

// ------------------------------------------------------------------ errors --
void set_error(const std::string &msg);
wr_status fail(wr_status code, const std::string &msg);

struct CudaError {
    wr_status code;
};

#define WR_CUDA(call)                                                            \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            ::wr::set_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
            throw ::wr::CudaError{e_ == cudaErrorMemoryAllocation ? WR_ENOMEM : WR_ECUDA}; \
        }                                                                        \
    } while (0)

#define WR_LAUNCH_CHECK() WR_CUDA(cudaGetLastError())

struct Status {
    wr_status code;
    std::string msg;
};
#define WR_THROW(code, msg) throw ::wr::Status{(code), (msg)}

// Runs f() translating exceptions into wr_status + wr_last_error().
template <class F>
wr_status guarded(F &&f) {
    try {
        return f();
    } catch (const CudaError &e) {
        return e.code;
    } catch (const Status &s) {
        return fail(s.code, s.msg);
    } catch (const std::bad_alloc &) {
        return fail(WR_ENOMEM, "host allocation failed");
    } catch (...) {
        return fail(WR_EINTERNAL, "unexpected exception");
    }
}

// NVTX range for the lifetime of a scope (tracing, §5): every entry point
// and the sweep / pred / route phases (header-only NVTX v3).
struct NvtxRange {
    explicit NvtxRange(const char *name);
    ~NvtxRange();
};

// Counts libwr kernel launches (reported in stats and by the bench).
extern thread_local int64_t g_launches;
inline void count_launch() { ++g_launches; }

// --------------------------------------------------------- device memory --
// Stream-ordered allocations from a per-device memory pool that keeps freed
// blocks reserved (release threshold = max), so a steady stream of calls
// (the bench, a serving loop) does not pay cudaMalloc/cudaFree of the
// multi-GB Bellman-Ford working set on every call. Each API entry point sets
// the calling thread's stream (StreamScope); buffers are allocated and freed
// in that stream's order.
extern thread_local cudaStream_t g_stream;
void *pool_alloc(size_t bytes, cudaStream_t s);
void pool_free(void *p, cudaStream_t s);
// Bytes reserved by the pool but not in use (reusable by the next call).
size_t pool_idle_bytes(int device);

struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(g_stream) { g_stream = s; }
    ~StreamScope() { g_stream = prev; }
};

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count == 0) return;
        s = g_stream;
        p = (T *)pool_alloc(count * sizeof(T), s);
        n = count;
    }
    void release() {
        if (p) pool_free(p, s);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// True if ptr is device (or managed) memory usable by kernels.
bool is_device_ptr(const void *ptr);

// Copies a caller array (host or device) into a fresh device buffer.
template <class T>
DBuf<T> to_device(const T *src, size_t count, cudaStream_t st) {
    DBuf<T> d(count);
    if (count) WR_CUDA(cudaMemcpyAsync(d.p, src, count * sizeof(T), cudaMemcpyDefault, st));
    return d;
}

// ------------------------------------------------------------ the graph --
struct DevGraph {           // kernel view (POD)
    int V;
    int E;
    const int *in_ptr;      // [V+1] CSC offsets (in-arcs of v)
    const int *in_src;      // [E]   tail u of each in-arc, sorted by (v, u)
    const uint32_t *in_w;   // [E]   weight bits
    const int2 *in_arc;     // [E]   (in_src, in_w) packed: one 8-B load per in-arc
    const int *out_ptr;     // [V+1] CSR offsets (out-arcs of u)
    const int *out_dst;     // [E]   head of each out-arc
};

}  // namespace wr

struct wr_graph {
    int device = 0;
    int V = 0;
    int64_t E = 0;
    int wtype = WR_I32;
    int has_negative = 0;
    int has_zero = 0;       // an int32 arc of weight 0
    int32_t max_abs_w = 0;
    int64_t max_in_deg = 0; // largest in-degree (keyed rows need <= 15)
    float max_w_f = 0.f;    // fp32 graphs: largest weight (near-far threshold step)
    wr::DBuf<int> in_ptr, in_src, out_ptr, out_dst;
    wr::DBuf<uint32_t> in_w;
    wr::DBuf<int2> in_arc;
    wr::DBuf<int> xy;       // [V*2] or empty
    wr::DBuf<int> z;        // [V] rack level or empty
    mutable wr::DBuf<int> hop_c;  // [V] BFS hops from a central vertex (tile cost key), built on first use
    int bbox[6] = {0, 0, 0, 0, 0, 0};   // xmin, xmax, ymin, ymax, zmin, zmax
    wr::DevGraph view() const {
        return wr::DevGraph{V, (int)E, in_ptr.p, in_src.p, in_w.p, in_arc.p, out_ptr.p, out_dst.p};
    }
};

namespace wr {

// --------------------------------------------------------- scan helpers --
// Exclusive prefix sum of n int64 values (device in/out may alias).
void scan_exclusive_i64(const int64_t *in, int64_t *out, int64_t n, cudaStream_t st);
void scan_exclusive_i32(const int *in, int *out, int n, cudaStream_t st);

// -------------------------------------------------------- Bellman-Ford --
// Segment scheduler (a8): sources per BF batch for a per-source byte cost.
int64_t budget_bytes(int64_t requested, int64_t fixed, int64_t want_pooled);
int64_t sources_per_segment(int64_t budget, int64_t fixed_bytes, int64_t per_source_bytes,
                            int64_t S, int tsw);
// Sources per lane (1, 2, 4) for S sources on nsm SMs (env WR_BF_SPL forces).
int choose_spl(int64_t S, int nsm, int pack);
// Near-far threshold step for an fp32 graph (0 = off): WR_NF_DELTA x the
// largest weight (default measured).
float nf_delta_for(const wr_graph *g);

// The canonical-pred pass fused into the sweep: CTAs whose tile claims have
// run out take pred jobs of finished tiles (in completion order) while the
// last tiles are still relaxing (a4 overlapped with the a3 tail).
struct PredFuse {
    int32_t *pred_out = nullptr;    // null = no fused pred
    int64_t out_row0 = 0;
    int *flat_tiles = nullptr;      // [ntiles] set if a tile has a flat vertex
    int *done_list = nullptr;       // [ntiles] finished tiles in completion order, -1 = not yet
    int *counters = nullptr;        // [4] zeroed: [0] done slots, [2..3] u64 pred jobs claimed
    long long *trace = nullptr;     // diagnostics (WR_TILE_TRACE): per tile {start, end, rounds, SM}
};

// NEXT-3 near-far (§1.1 leaves Δ-stepping
// for future work): a vertex improved to a distance beyond the tile's
// threshold T (all improved slots > T) keeps its new row but defers its
// propagation (no change bit, no out-neighbour marks) until T reaches it;
// T grows by delta per round, and jumps to the nearest deferred key when a
// round has nothing near. Per persistent CTA: keys[V] (min deferred key),
// plist[2][ceil(V/32)] (words with deferred vertices, double-buffered).
struct NearFar {
    uint32_t *keys = nullptr;   // gridDim.x x V
    int *plist = nullptr;       // gridDim.x x 2 x NW
    float delta = 0.f;          // 0 = off
};

struct BfRun {              // one BF segment over tiles of 32*spl sources
    const int *tile_src;    // [ntiles*tsw] source vertex per slot, -1 = empty
    int ntiles;
    uint32_t *rows;         // [ntiles][V][tsw] working distances (output)
    int variant;
    int max_rounds;
    int spl;                // 32-bit words per lane; a row has 32*spl words
    const int *slot_row = nullptr;  // [ntiles*tsw] output row offset per slot (null = identity)
    int pack = 1;           // sources per 32-bit word: 1, or 2 (packed u16 distances)
    const int *tile_order = nullptr;  // [ntiles] claim order of the tiles (null = 0..ntiles-1)
    uint32_t ovf_thr = 0;   // pack 2: a stored distance >= ovf_thr flags a possible u16 overflow
    bool keyed = false;     // pack 2 rows hold (d << 4 | in-arc index of the pred) keys (OpK16)
    float nf_delta = 0.f;   // > 0: near-far deferral (fp32 rows), NearFar above
    PredFuse fuse;
    int tsw() const { return 32 * spl * pack; }   // sources (slots) per tile
};

struct BfTileStats {        // per-call accumulators (device)
    unsigned long long relax;
    int rounds_max;
    int negcycle_tile;      // -1 or a tile with a negative cycle
    unsigned long long visits;  // candidate (vertex, round) visits
    int overflow;           // pack 2: a stored distance reached ovf_thr (redo with 32-bit rows)
};

// Launches the relaxation sweep of a segment on stream st (a3).
void bf_run(const wr_graph *g, const BfRun &run, BfTileStats *d_stats, cudaStream_t st);

// Canonical pred (a4) + output of dist/pred rows of a segment in S x T /
// S x V row-major caller layout, row index = out_row0 + tile*32 + lane.
void bf_write_outputs(const wr_graph *g, const BfRun &run, int64_t out_row0, int64_t S_total,
                      const int *targets, int T, void *dist_out, int32_t *pred_out,
                      int *d_flat_tiles, cudaStream_t st);
// Resolves "flat" predecessors of the listed tiles with a tight-arc BFS.
// gate: optional device [ntiles] flags; a listed tile whose flag is 0 is
// skipped on the device (no host readback needed).
void bf_resolve_flat(const wr_graph *g, const BfRun &run, const std::vector<int> &tiles,
                     int64_t out_row0, int32_t *pred_out, cudaStream_t st, const int *gate = nullptr);

// Builds the tiles for sources [lo, hi) of a device source list: tsw slots
// per tile, spatially compact (recursive coordinate bisection of the
// graph's coordinates when present), ceil(n / tsw) full tiles (or, with
// WR_TILE_BALANCE, a whole number of waves of tiles <= max_tiles):
// tile_src[slot] = source vertex, slot_row[slot] = source offset in
// [0, hi-lo) (-1 = empty slot), pos_of[offset] = slot position. Returns the
// number of tiles (wr_tiles.cu).
int make_tiles_ordered(const wr_graph *g, const int *d_sources, int64_t lo, int64_t hi, int tsw, int64_t max_tiles,
                       int *tile_src, int *slot_row, int *pos_of, cudaStream_t st);
// Tiles to allocate for segments of sb sources: sb/tsw (with WR_TILE_BALANCE
// plus up to one wave of extra, partly filled tiles if extra_bytes allow).
int64_t tiles_to_allocate(int64_t sb, int tsw, int64_t extra_bytes, int64_t tile_bytes);

// ------------------------------------------------------------- routing --
struct RouteProblem {       // one exhaustive search (an order or a segment)
    int order;              // index into the D array
    int n;                  // stops in this problem (<= WR_MAX_EXACT)
    int dep;                // -1 open; else the order-stop index of the depot (closed tour, NEXT-4)
    uint64_t map;           // 4-bit local -> order-stop index, position k at bits 4k
    int item0;              // first work item
    int nitems;
};

struct RouteWorkItem {
    int problem;
    int prefix_lo;          // first prefix (lexicographic) of this chunk
    int prefix_hi;
};

// Prefix depth p(n) used to split n! into subtrees of (n-p)! leaves.
int route_prefix_depth(int n);
int64_t factorial64(int n);

}  // namespace wr
