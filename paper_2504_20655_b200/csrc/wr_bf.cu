// wr_bf.cu - a3 batched Bellman-Ford relaxation sweep, a4 canonical
// predecessor, a8 source-batch scheduler, and the wr_bf_batch entry point.
//
// The paper's kernel (P720-724 §4.7) is edge-parallel, one thread per edge,
// (V-1) rounds with a host sync per round, dist/pred V x N in global memory
// with write contention. This design is B200-first instead:
//   * sources are the SIMD lanes: a tile of 32 sources is one 128-byte row
//     per vertex (rows[tile][v][lane]); every neighbour gather is one fully
//     coalesced 128-B line and the graph arc (u, w) is loaded once per 32
//     relaxations;
//   * one CTA owns a tile and iterates its rounds alone (no grid sync, no
//     host sync per round - the paper's 10.3 us/round), tiles are claimed
//     from a persistent work counter;
//   * frontier pull: a round relaxes only vertices with an in-neighbour that
//     changed in the previous round (bitmaps in shared memory, expanded over
//     the CSR out-arcs); the change mask of a vertex is one __any_sync vote;
//   * atomic-free commit: each (v, lane) has exactly one writer (the warp
//     that owns v's candidate word), updates are in place (chaotic /
//     Gauss-Seidel), which reaches the same unique fixpoint (reading O2:
//     the relaxation operator is monotone and deflationary for w >= 0, and
//     exact for int weights), so dist is bit-identical to the oracle;
//   * pred is not written inside the racy sweep: a4 recomputes the
//     canonical predecessor from the converged dist (O3), deterministic.
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "wr_internal.cuh"

namespace wr {

constexpr int TS = 32;          // sources per tile (lanes)
constexpr int BF_THREADS = 512; // 16 warps per CTA

// ------------------------------------------------------------- weight ops --
// Nonnegative int32: unsigned add + min (DPX VIADDMNMX). INF = INT32_MAX, and
// INF + w (w < 2^31) never wraps and never beats a finite value: an INF tail
// relaxes nothing, exactly like the oracle's "skip d[u] == INF".
struct OpU32 {
    static constexpr uint32_t INF = 0x7fffffffu;
    static constexpr uint32_t ZERO = 0u;
    __device__ __forceinline__ static uint32_t relax(uint32_t d, uint32_t du, uint32_t w) {
        return __viaddmin_u32(du, w, d);
    }
    __device__ __forceinline__ static bool less(uint32_t a, uint32_t b) { return a < b; }
    __device__ __forceinline__ static bool finite(uint32_t x) { return x != INF; }
    __device__ __forceinline__ static bool tight(uint32_t du, uint32_t w, uint32_t dv) {
        return du != INF && du + w == dv;
    }
};
// fp32 (weights finite, >= 0): one IEEE binary32 RN add, then min. +inf
// tails give +inf, which never wins.
struct OpF32 {
    static constexpr uint32_t INF = 0x7f800000u;
    static constexpr uint32_t ZERO = 0u;
    __device__ __forceinline__ static uint32_t relax(uint32_t d, uint32_t du, uint32_t w) {
        const float c = __fadd_rn(__uint_as_float(du), __uint_as_float(w));
        return c < __uint_as_float(d) ? __float_as_uint(c) : d;
    }
    __device__ __forceinline__ static bool less(uint32_t a, uint32_t b) {
        return __uint_as_float(a) < __uint_as_float(b);
    }
    __device__ __forceinline__ static bool finite(uint32_t x) { return x != INF; }
    __device__ __forceinline__ static bool tight(uint32_t du, uint32_t w, uint32_t dv) {
        return du != INF && __fadd_rn(__uint_as_float(du), __uint_as_float(w)) == __uint_as_float(dv);
    }
};
// int32 with negative weights: exact 64-bit candidate, INF tails skipped.
struct OpI32N {
    static constexpr uint32_t INF = 0x7fffffffu;
    static constexpr uint32_t ZERO = 0u;
    __device__ __forceinline__ static uint32_t relax(uint32_t d, uint32_t du, uint32_t w) {
        if (du == INF) return d;
        const int64_t c = (int64_t)(int)du + (int64_t)(int)w;
        return c < (int64_t)(int)d ? (uint32_t)(int)c : d;
    }
    __device__ __forceinline__ static bool less(uint32_t a, uint32_t b) { return (int)a < (int)b; }
    __device__ __forceinline__ static bool finite(uint32_t x) { return x != INF; }
    __device__ __forceinline__ static bool tight(uint32_t du, uint32_t w, uint32_t dv) {
        return du != INF && (int64_t)(int)du + (int64_t)(int)w == (int64_t)(int)dv;
    }
};

// ------------------------------------------------------------ tile setup --
__global__ void make_tiles_kernel(const int *sources, int64_t lo, int64_t hi, int *tile_src, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    tile_src[i] = (lo + i < hi) ? sources[lo + i] : -1;
}

void make_tiles(const int *d_sources, int64_t lo, int64_t hi, int *d_tile_src, cudaStream_t st) {
    const int64_t ntiles = (hi - lo + TS - 1) / TS;
    const int64_t n = ntiles * TS;
    if (n == 0) return;
    make_tiles_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_sources, lo, hi, d_tile_src, n);
    count_launch();
    WR_LAUNCH_CHECK();
}

// ---------------------------------------------------- relaxing one word --
constexpr uint32_t FULL = 0xffffffffu;

// Pull over all in-arcs of v for the 32 lanes (generic degree).
template <class Op>
__device__ __forceinline__ uint32_t relax_vertex(const DevGraph &g, const uint32_t *__restrict__ R, int a0, int a1,
                                                 int lane, uint32_t d) {
    for (int base = a0; base < a1; base += 32) {
        const int cnt = min(32, a1 - base);
        int my_u = 0;
        uint32_t my_w = 0;
        if (lane < cnt) {
            my_u = g.in_src[base + lane];
            my_w = g.in_w[base + lane];
        }
        int k = 0;
        for (; k + 4 <= cnt; k += 4) {
            const int u0 = __shfl_sync(FULL, my_u, k), u1 = __shfl_sync(FULL, my_u, k + 1);
            const int u2 = __shfl_sync(FULL, my_u, k + 2), u3 = __shfl_sync(FULL, my_u, k + 3);
            const uint32_t w0 = __shfl_sync(FULL, my_w, k), w1 = __shfl_sync(FULL, my_w, k + 1);
            const uint32_t w2 = __shfl_sync(FULL, my_w, k + 2), w3 = __shfl_sync(FULL, my_w, k + 3);
            const uint32_t x0 = R[(size_t)u0 * TS + lane], x1 = R[(size_t)u1 * TS + lane];
            const uint32_t x2 = R[(size_t)u2 * TS + lane], x3 = R[(size_t)u3 * TS + lane];
            d = Op::relax(d, x0, w0);
            d = Op::relax(d, x1, w1);
            d = Op::relax(d, x2, w2);
            d = Op::relax(d, x3, w3);
        }
        for (; k < cnt; ++k) {
            const int u = __shfl_sync(FULL, my_u, k);
            const uint32_t wk = __shfl_sync(FULL, my_w, k);
            d = Op::relax(d, R[(size_t)u * TS + lane], wk);
        }
    }
    return d;
}

// Relaxes the candidate vertices (bits of m) of word w for all 32 lanes.
// The word's CSC offsets are read with one coalesced load; two candidates
// are processed per iteration (lanes 0-15 hold the first one's arcs, 16-31
// the second's) so four independent 128-B row gathers are in flight.
// Returns the word's change mask (one __any_sync vote per vertex).
template <class Op>
__device__ __forceinline__ uint32_t relax_word(const DevGraph &g, uint32_t *__restrict__ R, int w, uint32_t m,
                                               int lane, unsigned long long &relax) {
    const int vl = (w << 5) + lane;
    int p_lo = 0, p_hi = 0;
    if (vl < g.V) {
        p_lo = g.in_ptr[vl];
        p_hi = g.in_ptr[vl + 1];
    }
    uint32_t chg = 0;
    while (m) {
        const int b0 = __ffs(m) - 1;
        m &= m - 1;
        const bool two = m != 0;
        int b1 = b0;
        if (two) {
            b1 = __ffs(m) - 1;
            m &= m - 1;
        }
        const int v0 = (w << 5) + b0, v1 = (w << 5) + b1;
        const int a00 = __shfl_sync(FULL, p_lo, b0), a01 = __shfl_sync(FULL, p_hi, b0);
        const int a10 = __shfl_sync(FULL, p_lo, b1), a11 = __shfl_sync(FULL, p_hi, b1);
        const int n0 = a01 - a00, n1 = two ? a11 - a10 : 0;
        const uint32_t e0 = R[(size_t)v0 * TS + lane];
        const uint32_t e1 = two ? R[(size_t)v1 * TS + lane] : 0u;
        uint32_t d0 = e0, d1 = e1;
        if (n0 <= 16 && n1 <= 16) {
            const int sub = lane & 15;
            const int base = lane < 16 ? a00 : a10;
            const int cnt = lane < 16 ? n0 : n1;
            int my_u = 0;
            uint32_t my_w = 0;
            if (sub < cnt) {
                my_u = g.in_src[base + sub];
                my_w = g.in_w[base + sub];
            }
            const int kmax = max(n0, n1);
            for (int k = 0; k < kmax; k += 2) {
                const int u00 = __shfl_sync(FULL, my_u, k), u01 = __shfl_sync(FULL, my_u, k + 1);
                const int u10 = __shfl_sync(FULL, my_u, 16 + k), u11 = __shfl_sync(FULL, my_u, 17 + k);
                const uint32_t w00 = __shfl_sync(FULL, my_w, k), w01 = __shfl_sync(FULL, my_w, k + 1);
                const uint32_t w10 = __shfl_sync(FULL, my_w, 16 + k), w11 = __shfl_sync(FULL, my_w, 17 + k);
                const uint32_t x00 = k < n0 ? R[(size_t)u00 * TS + lane] : 0u;
                const uint32_t x01 = k + 1 < n0 ? R[(size_t)u01 * TS + lane] : 0u;
                const uint32_t x10 = k < n1 ? R[(size_t)u10 * TS + lane] : 0u;
                const uint32_t x11 = k + 1 < n1 ? R[(size_t)u11 * TS + lane] : 0u;
                if (k < n0) d0 = Op::relax(d0, x00, w00);
                if (k + 1 < n0) d0 = Op::relax(d0, x01, w01);
                if (k < n1) d1 = Op::relax(d1, x10, w10);
                if (k + 1 < n1) d1 = Op::relax(d1, x11, w11);
            }
        } else {
            d0 = relax_vertex<Op>(g, R, a00, a01, lane, d0);
            if (two) d1 = relax_vertex<Op>(g, R, a10, a11, lane, d1);
        }
        relax += (unsigned long long)(n0 + n1);
        const bool c0 = Op::less(d0, e0);
        if (c0) R[(size_t)v0 * TS + lane] = d0;
        if (__any_sync(FULL, c0)) chg |= 1u << b0;
        if (two) {
            const bool c1 = Op::less(d1, e1);
            if (c1) R[(size_t)v1 * TS + lane] = d1;
            if (__any_sync(FULL, c1)) chg |= 1u << b1;
        }
    }
    return chg;
}

// ------------------------------------------------------ the sweep kernel --
// One CTA per tile at a time. Shared memory: two V-bit bitmaps
// (changed = vertices improved last round, cand = their out-neighbours).
template <class Op, bool DENSE>
__global__ void __launch_bounds__(BF_THREADS) bf_frontier_kernel(DevGraph g, const int *__restrict__ tile_src,
                                                                 int ntiles, uint32_t *__restrict__ rows,
                                                                 int *tile_counter, int max_rounds,
                                                                 BfTileStats *stats) {
    extern __shared__ uint32_t smem[];
    const int V = g.V;
    const int NW = (V + 31) >> 5;
    uint32_t *changed = smem;
    uint32_t *cand = smem + NW;
    __shared__ int s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWARPS = BF_THREADS / 32;
    const uint32_t last_mask = (V & 31) ? ((1u << (V & 31)) - 1u) : 0xffffffffu;

    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
        __syncthreads();
        const int tile = s_tile;
        if (tile >= ntiles) break;
        uint32_t *R = rows + (size_t)tile * V * TS;

        // init: every row INF, bitmaps empty
        {
            uint4 inf4 = make_uint4(Op::INF, Op::INF, Op::INF, Op::INF);
            uint4 *R4 = reinterpret_cast<uint4 *>(R);
            const size_t n4 = (size_t)V * (TS / 4);
            for (size_t i = threadIdx.x; i < n4; i += BF_THREADS) R4[i] = inf4;
            for (int w = threadIdx.x; w < NW; w += BF_THREADS) {
                changed[w] = 0u;
                cand[w] = 0u;
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int s = tile_src[tile * TS + lane];
            if (s >= 0) {
                R[(size_t)s * TS + lane] = Op::ZERO;
                atomicOr(&changed[s >> 5], 1u << (s & 31));
            }
        }
        __syncthreads();

        int rounds = 0;
        unsigned long long relax = 0;
        bool more = true;
        while (more) {
            // ---- expand: cand = out-neighbours of changed (dense: all)
            if (DENSE) {
                for (int w = threadIdx.x; w < NW; w += BF_THREADS) {
                    cand[w] = (w == NW - 1) ? last_mask : 0xffffffffu;
                    changed[w] = 0u;
                }
            } else {
                for (int w = threadIdx.x; w < NW; w += BF_THREADS) {
                    uint32_t m = changed[w];
                    if (!m) continue;
                    changed[w] = 0u;
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        const int u = (w << 5) + b;
                        const int e1 = g.out_ptr[u + 1];
                        for (int e = g.out_ptr[u]; e < e1; ++e) {
                            const int x = g.out_dst[e];
                            atomicOr(&cand[x >> 5], 1u << (x & 31));
                        }
                    }
                }
            }
            __syncthreads();
            // ---- relax: warp per candidate word, lane = source
            int any = 0;
            for (int w = warp; w < NW; w += NWARPS) {
                uint32_t m = cand[w];
                if (!m) continue;
                __syncwarp();
                if (lane == 0) cand[w] = 0u;
                const uint32_t chg = relax_word<Op>(g, R, w, m, lane, relax);
                if (chg) {
                    if (lane == 0) changed[w] = chg;
                    any = 1;
                }
            }
            ++rounds;
            more = __syncthreads_or(any) != 0;
            if (more && rounds >= max_rounds) {
                if (threadIdx.x == 0) atomicMax(&stats->negcycle_tile, tile);
                more = false;
            }
        }
        // per-tile statistics (one lane per warp contributes its arc count)
        if (lane == 0 && relax) atomicAdd(&stats->relax, relax * TS);
        if (threadIdx.x == 0) atomicMax(&stats->rounds_max, rounds);
        __syncthreads();
    }
}

template <class Op>
static void launch_sweep(const wr_graph *g, const BfRun &run, BfTileStats *d_stats, cudaStream_t st) {
    const int V = g->V;
    const int NW = (V + 31) / 32;
    const size_t smem = (size_t)2 * NW * sizeof(uint32_t);
    int dev = g->device;
    int max_optin = 0;
    WR_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (smem + 1024 > (size_t)max_optin)
        WR_THROW(WR_ETOOLARGE, "bf: V too large for the shared-memory frontier bitmaps");
    auto kern = run.variant == WR_BF_DENSE ? bf_frontier_kernel<Op, true> : bf_frontier_kernel<Op, false>;
    WR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, nsm = 0;
    WR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BF_THREADS, smem));
    WR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    per_sm = std::max(per_sm, 1);
    const int grid = std::min<int64_t>(run.ntiles, (int64_t)per_sm * nsm);
    DBuf<int> counter(1);
    WR_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(int), st));
    kern<<<grid, BF_THREADS, smem, st>>>(g->view(), run.tile_src, run.ntiles, run.rows, counter.p,
                                         run.max_rounds, d_stats);
    count_launch();
    WR_LAUNCH_CHECK();
    WR_CUDA(cudaStreamSynchronize(st));  // counter lifetime
}

void bf_run(const wr_graph *g, const BfRun &run, BfTileStats *d_stats, cudaStream_t st) {
    if (run.ntiles <= 0) return;
    if (g->wtype == WR_F32) launch_sweep<OpF32>(g, run, d_stats, st);
    else if (g->has_negative) launch_sweep<OpI32N>(g, run, d_stats, st);
    else launch_sweep<OpU32>(g, run, d_stats, st);
}

// --------------------------------------------------- a4 + output layout --
// Block = 8 warps; warp handles 32 consecutive output columns (vertices or
// targets) of one tile: computes dist/pred for (column j, lane = source k),
// stages them in shared memory and writes each source's 32 columns as one
// coalesced 128-B segment of the caller's row-major S x T / S x V arrays.
// Canonical pred (O3, w >= 0): smallest tail of a steep tight in-arc; a
// reachable non-source vertex without one is "flat" and is resolved by
// bf_resolve_flat. Graphs with a negative weight resolve every vertex there.
constexpr int OUT_WARPS = 4;
template <class Op>
__global__ void __launch_bounds__(OUT_WARPS * 32) bf_outputs_kernel(DevGraph g, const int *__restrict__ tile_src,
                                                         int ntiles, const uint32_t *__restrict__ rows,
                                                         int64_t out_row0, const int *__restrict__ targets,
                                                         int T, uint32_t *dist_out, int32_t *pred_out,
                                                         int *flat_tiles, int neg_graph) {
    __shared__ uint32_t sd[OUT_WARPS][32][33];
    __shared__ int32_t sp[OUT_WARPS][32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int V = g.V;
    const int ncols = targets ? T : V;
    const int chunks = (ncols + 31) / 32;
    const int64_t job = (int64_t)blockIdx.x * OUT_WARPS + warp;
    if (job >= (int64_t)ntiles * chunks) return;
    const int tile = (int)(job / chunks);
    const int c0 = (int)(job % chunks) * 32;
    const uint32_t *R = rows + (size_t)tile * V * TS;
    const int s = tile_src[tile * TS + lane];
    bool flat = false;
    for (int j = 0; j < 32; ++j) {
        const int col = c0 + j;
        if (col >= ncols) break;
        const int v = targets ? targets[col] : col;
        const uint32_t d = R[(size_t)v * TS + lane];
        sd[warp][j][lane] = d;
        if (pred_out && !targets) {
            // lane-divergent predicate; the shuffles below stay warp-uniform
            const bool active = v != s && s >= 0 && Op::finite(d);
            int best = 0x7fffffff;
            if (!neg_graph) {
                const int a0 = g.in_ptr[v], a1 = g.in_ptr[v + 1];
                for (int base = a0; base < a1; base += 32) {
                    const int cnt = min(32, a1 - base);
                    int my_u = 0;
                    uint32_t my_w = 0;
                    if (lane < cnt) {
                        my_u = g.in_src[base + lane];
                        my_w = g.in_w[base + lane];
                    }
                    for (int k = 0; k < cnt; ++k) {
                        const int u = __shfl_sync(0xffffffffu, my_u, k);
                        const uint32_t wk = __shfl_sync(0xffffffffu, my_w, k);
                        const uint32_t du = R[(size_t)u * TS + lane];
                        if (active && Op::tight(du, wk, d) && Op::less(du, d) && u < best) best = u;
                    }
                }
            }
            int p = -1;
            if (active) {
                if (best != 0x7fffffff) p = best;
                else flat = true;   // resolved by the tight-arc BFS pass
            }
            sp[warp][j][lane] = p;
        }
    }
    __syncwarp();
    // write out: for each source row k, columns c0..c0+31 (lane = column)
    const int col = c0 + lane;
    for (int k = 0; k < TS; ++k) {
        const int sk = tile_src[tile * TS + k];
        if (sk < 0) break;                       // tiles are filled lane 0 first
        const int64_t row = out_row0 + (int64_t)tile * TS + k;
        if (col < ncols) {
            if (dist_out) dist_out[row * ncols + col] = sd[warp][lane][k];
            if (pred_out && !targets) pred_out[row * (int64_t)V + col] = sp[warp][lane][k];
        }
    }
    if (__any_sync(0xffffffffu, flat) && lane == 0) atomicOr(&flat_tiles[tile], 1);
}

void bf_write_outputs(const wr_graph *g, const BfRun &run, int64_t out_row0, int64_t, const int *targets,
                      int T, void *dist_out, int32_t *pred_out, int *d_flat_tiles, cudaStream_t st) {
    if (run.ntiles <= 0 || (!dist_out && !pred_out)) return;
    const int ncols = targets ? T : g->V;
    const int64_t jobs = (int64_t)run.ntiles * ((ncols + 31) / 32);
    const unsigned grid = (unsigned)((jobs + OUT_WARPS - 1) / OUT_WARPS);
    const int neg = g->has_negative;
    if (g->wtype == WR_F32)
        bf_outputs_kernel<OpF32><<<grid, OUT_WARPS * 32, 0, st>>>(g->view(), run.tile_src, run.ntiles, run.rows, out_row0,
                                                       targets, T, (uint32_t *)dist_out, pred_out,
                                                       d_flat_tiles, neg);
    else if (neg)
        bf_outputs_kernel<OpI32N><<<grid, OUT_WARPS * 32, 0, st>>>(g->view(), run.tile_src, run.ntiles, run.rows, out_row0,
                                                        targets, T, (uint32_t *)dist_out, pred_out,
                                                        d_flat_tiles, neg);
    else
        bf_outputs_kernel<OpU32><<<grid, OUT_WARPS * 32, 0, st>>>(g->view(), run.tile_src, run.ntiles, run.rows, out_row0,
                                                       targets, T, (uint32_t *)dist_out, pred_out,
                                                       d_flat_tiles, neg);
    count_launch();
    WR_LAUNCH_CHECK();
}

// --------------------------------------------- flat predecessors (rare) --
// hop[v][k] = BFS layer of v over the tight arcs of source k (a min-plus
// sweep with unit weights restricted to tight arcs), then for every flat
// (v, k) - or every reachable vertex of a negative-weight graph -
// pred = argmin over tight in-arcs of (hop[u], u)  (O3).
template <class Op>
__global__ void __launch_bounds__(BF_THREADS) hop_bfs_kernel(DevGraph g, const int *__restrict__ tile_src,
                                                             int tile, const uint32_t *__restrict__ rows,
                                                             uint32_t *__restrict__ hop) {
    extern __shared__ uint32_t smem[];
    const int V = g.V;
    const int NW = (V + 31) >> 5;
    uint32_t *changed = smem;
    uint32_t *cand = smem + NW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWARPS = BF_THREADS / 32;
    const uint32_t *R = rows + (size_t)tile * V * TS;
    for (size_t i = threadIdx.x; i < (size_t)V * TS; i += BF_THREADS) hop[i] = 0xffffffffu;
    for (int w = threadIdx.x; w < NW; w += BF_THREADS) changed[w] = cand[w] = 0u;
    __syncthreads();
    if (warp == 0) {
        const int s = tile_src[tile * TS + lane];
        if (s >= 0) {
            hop[(size_t)s * TS + lane] = 0;
            atomicOr(&changed[s >> 5], 1u << (s & 31));
        }
    }
    __syncthreads();
    bool more = true;
    while (more) {
        for (int w = threadIdx.x; w < NW; w += BF_THREADS) {
            uint32_t m = changed[w];
            if (!m) continue;
            changed[w] = 0u;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int u = (w << 5) + b;
                for (int e = g.out_ptr[u]; e < g.out_ptr[u + 1]; ++e) {
                    const int x = g.out_dst[e];
                    atomicOr(&cand[x >> 5], 1u << (x & 31));
                }
            }
        }
        __syncthreads();
        int any = 0;
        for (int w = warp; w < NW; w += NWARPS) {
            uint32_t m = cand[w];
            if (!m) continue;
            __syncwarp();
            if (lane == 0) cand[w] = 0u;
            uint32_t chg = 0;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int v = (w << 5) + b;
                const uint32_t dv = R[(size_t)v * TS + lane];
                const uint32_t h0 = hop[(size_t)v * TS + lane];
                uint32_t h = h0;
                for (int e = g.in_ptr[v]; e < g.in_ptr[v + 1]; ++e) {
                    const int u = g.in_src[e];
                    const uint32_t hu = hop[(size_t)u * TS + lane];
                    if (hu != 0xffffffffu && Op::tight(R[(size_t)u * TS + lane], g.in_w[e], dv) && hu + 1 < h)
                        h = hu + 1;
                }
                const bool c = h < h0;
                if (c) hop[(size_t)v * TS + lane] = h;
                if (__any_sync(0xffffffffu, c)) chg |= 1u << b;
            }
            if (chg) {
                if (lane == 0) changed[w] = chg;
                any = 1;
            }
        }
        more = __syncthreads_or(any) != 0;
    }
}

template <class Op>
__global__ void flat_pred_kernel(DevGraph g, const int *__restrict__ tile_src, int tile,
                                 const uint32_t *__restrict__ rows, const uint32_t *__restrict__ hop,
                                 int64_t out_row0, int32_t *pred_out, int neg_graph) {
    const int lane = threadIdx.x & 31;
    const int v = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int V = g.V;
    if (v >= V) return;
    const uint32_t *R = rows + (size_t)tile * V * TS;
    const int s = tile_src[tile * TS + lane];
    const uint32_t d = R[(size_t)v * TS + lane];
    if (s < 0 || v == s || !Op::finite(d)) return;
    bool steep = false;
    int best = -1;
    uint32_t best_h = 0xffffffffu;
    for (int e = g.in_ptr[v]; e < g.in_ptr[v + 1]; ++e) {
        const int u = g.in_src[e];
        const uint32_t du = R[(size_t)u * TS + lane];
        if (!Op::tight(du, g.in_w[e], d)) continue;
        if (Op::less(du, d)) steep = true;
        const uint32_t hu = hop[(size_t)u * TS + lane];
        if (hu < best_h || (hu == best_h && u < best)) {
            best_h = hu;
            best = u;
        }
    }
    if (neg_graph || !steep) pred_out[(out_row0 + (int64_t)tile * TS + lane) * V + v] = best;
}

void bf_resolve_flat(const wr_graph *g, const BfRun &run, const std::vector<int> &tiles, int64_t out_row0,
                     int32_t *pred_out, cudaStream_t st) {
    if (tiles.empty() || !pred_out) return;
    const int V = g->V;
    DBuf<uint32_t> hop((size_t)V * TS);
    const size_t smem = (size_t)2 * ((V + 31) / 32) * sizeof(uint32_t);
    for (int t : tiles) {
        if (g->wtype == WR_F32) {
            WR_CUDA(cudaFuncSetAttribute(hop_bfs_kernel<OpF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            hop_bfs_kernel<OpF32><<<1, BF_THREADS, smem, st>>>(g->view(), run.tile_src, t, run.rows, hop.p);
            flat_pred_kernel<OpF32><<<(V + 7) / 8, 256, 0, st>>>(g->view(), run.tile_src, t, run.rows, hop.p,
                                                                 out_row0, pred_out, 0);
        } else if (g->has_negative) {
            WR_CUDA(cudaFuncSetAttribute(hop_bfs_kernel<OpI32N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            hop_bfs_kernel<OpI32N><<<1, BF_THREADS, smem, st>>>(g->view(), run.tile_src, t, run.rows, hop.p);
            flat_pred_kernel<OpI32N><<<(V + 7) / 8, 256, 0, st>>>(g->view(), run.tile_src, t, run.rows, hop.p,
                                                                  out_row0, pred_out, 1);
        } else {
            WR_CUDA(cudaFuncSetAttribute(hop_bfs_kernel<OpU32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            hop_bfs_kernel<OpU32><<<1, BF_THREADS, smem, st>>>(g->view(), run.tile_src, t, run.rows, hop.p);
            flat_pred_kernel<OpU32><<<(V + 7) / 8, 256, 0, st>>>(g->view(), run.tile_src, t, run.rows, hop.p,
                                                                 out_row0, pred_out, 0);
        }
        count_launch();
        count_launch();
        WR_LAUNCH_CHECK();
    }
    WR_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------ a8 the scheduler --
int64_t budget_bytes(int64_t requested) {
    size_t free_b = 0, total_b = 0;
    WR_CUDA(cudaMemGetInfo(&free_b, &total_b));
    int64_t b = requested > 0 ? requested : (int64_t)180e9;
    return std::min<int64_t>(b, (int64_t)(0.9 * (double)free_b));
}

int64_t sources_per_segment(int64_t budget, int64_t fixed_bytes, int64_t per_source_bytes, int64_t S) {
    const int64_t room = budget - fixed_bytes;
    if (room < per_source_bytes * TS)
        WR_THROW(WR_ENOMEM, "scheduler: HBM budget below one 32-source tile");
    int64_t sb = room / per_source_bytes;
    sb = (sb / TS) * TS;
    return std::max<int64_t>(TS, std::min<int64_t>(sb, ((S + TS - 1) / TS) * TS));
}

// ----------------------------------------------------- validation kernel --
__global__ void check_vertices_kernel(const int *v, int64_t n, int V, int *bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && (v[i] < 0 || v[i] >= V)) atomicOr(bad, 1);
}

static void check_vertices(const int *d_v, int64_t n, int V, cudaStream_t st, const char *what) {
    if (n <= 0) return;
    DBuf<int> bad(1);
    WR_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
    check_vertices_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_v, n, V, bad.p);
    count_launch();
    WR_LAUNCH_CHECK();
    int h = 0;
    WR_CUDA(cudaMemcpyAsync(&h, bad.p, 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    if (h) WR_THROW(WR_EINVAL, std::string(what) + ": vertex outside [0, V)");
}

// ------------------------------------------------------------ entry point --
static wr_status bf_batch_impl(const wr_graph *g, const int32_t *sources, int32_t S, const int32_t *targets,
                               int32_t T, void *dist, int32_t *pred, const wr_bf_opts *opts,
                               wr_bf_stats *stats) {
    if (!g) return fail(WR_EINVAL, "wr_bf_batch: null graph");
    if (S < 0 || (S > 0 && !sources)) return fail(WR_EINVAL, "wr_bf_batch: sources");
    if (targets && T < 0) return fail(WR_EINVAL, "wr_bf_batch: T");
    WR_CUDA(cudaSetDevice(g->device));
    const int64_t g_launch0 = g_launches;
    wr_bf_opts o{};
    if (opts) o = *opts;
    cudaStream_t st = (cudaStream_t)o.stream;
    const int V = g->V;
    const int ncols = targets ? T : V;
    int max_rounds = o.max_rounds > 0 ? o.max_rounds : std::max(1, V - 1);
    if (!g->has_negative && o.max_rounds <= 0) max_rounds = V;  // no negative cycle possible
    const int variant = o.variant == WR_BF_DENSE ? WR_BF_DENSE : WR_BF_FRONTIER;

    cudaEvent_t e0, e1;
    WR_CUDA(cudaEventCreate(&e0));
    WR_CUDA(cudaEventCreate(&e1));
    WR_CUDA(cudaEventRecord(e0, st));

    DBuf<int> d_src = to_device<int>(sources, S, st);
    check_vertices(d_src.p, S, V, st, "wr_bf_batch sources");
    DBuf<int> d_tgt;
    if (targets) {
        d_tgt = to_device<int>(targets, T, st);
        check_vertices(d_tgt.p, T, V, st, "wr_bf_batch targets");
    }
    const bool dist_dev = dist && is_device_ptr(dist);
    const bool pred_dev = pred && is_device_ptr(pred);

    // a8: per-source working set = rows (4V) + staging for host outputs
    int64_t per_src = 4LL * V;
    if (dist && !dist_dev) per_src += 4LL * ncols;
    if (pred && !pred_dev) per_src += 4LL * V;
    wr_graph_info_t gi;
    wr_graph_info(g, &gi);
    const int64_t budget = budget_bytes(o.hbm_budget);
    const int64_t sb = sources_per_segment(budget, gi.device_bytes + (64 << 20), per_src, std::max(S, 1));
    const int64_t max_tiles = sb / TS;

    DBuf<uint32_t> rows((size_t)max_tiles * V * TS);
    DBuf<int> tile_src(max_tiles * TS);
    DBuf<int> flat(max_tiles);
    DBuf<uint32_t> dist_stage;
    DBuf<int32_t> pred_stage;
    if (dist && !dist_dev) dist_stage.alloc((size_t)sb * ncols);
    if (pred && !pred_dev) pred_stage.alloc((size_t)sb * V);
    DBuf<BfTileStats> d_stats(1);
    BfTileStats h0{0ull, 0, -1};
    WR_CUDA(cudaMemcpyAsync(d_stats.p, &h0, sizeof(h0), cudaMemcpyHostToDevice, st));

    int segments = 0;
    int64_t total_tiles = 0;
    for (int64_t lo = 0; lo < S; lo += sb) {
        const int64_t hi = std::min<int64_t>(S, lo + sb);
        const int ntiles = (int)((hi - lo + TS - 1) / TS);
        make_tiles(d_src.p, lo, hi, tile_src.p, st);
        BfRun run{tile_src.p, ntiles, rows.p, variant, max_rounds};
        bf_run(g, run, d_stats.p, st);
        BfTileStats hs;
        WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
        if (hs.negcycle_tile >= 0) {
            int s_bad = -1;
            WR_CUDA(cudaMemcpy(&s_bad, tile_src.p + hs.negcycle_tile * TS, 4, cudaMemcpyDeviceToHost));
            if (stats) stats->negcycle_source = s_bad;
            if (g->has_negative && o.max_rounds <= 0)
                return fail(WR_ENEGCYCLE, "wr_bf_batch: negative cycle reachable from a source");
            return fail(WR_EINTERNAL, "wr_bf_batch: max_rounds reached before convergence");
        }
        uint32_t *dout = dist ? (dist_dev ? (uint32_t *)dist : dist_stage.p) : nullptr;
        int32_t *pout = pred ? (pred_dev ? pred : pred_stage.p) : nullptr;
        // device outputs are addressed with the caller's global row, staging
        // buffers with the row inside the segment
        const int64_t row_d = dist_dev ? lo : 0, row_p = pred_dev ? lo : 0;
        WR_CUDA(cudaMemsetAsync(flat.p, 0, sizeof(int) * ntiles, st));
        if (dout && pout && !targets && row_d == row_p) {
            bf_write_outputs(g, run, row_d, S, nullptr, V, dout, pout, flat.p, st);
        } else {
            if (dout) bf_write_outputs(g, run, row_d, S, d_tgt.p, ncols, dout, nullptr, flat.p, st);
            if (pout) bf_write_outputs(g, run, row_p, S, nullptr, V, nullptr, pout, flat.p, st);
        }
        if (pout) {
            std::vector<int> hflat(ntiles);
            WR_CUDA(cudaMemcpyAsync(hflat.data(), flat.p, sizeof(int) * ntiles, cudaMemcpyDeviceToHost, st));
            WR_CUDA(cudaStreamSynchronize(st));
            std::vector<int> todo;
            for (int t = 0; t < ntiles; ++t)
                if (hflat[t] || g->has_negative) todo.push_back(t);
            bf_resolve_flat(g, run, todo, pred_dev ? lo : 0, pout, st);
        }
        if (dist && !dist_dev)
            WR_CUDA(cudaMemcpyAsync((char *)dist + (size_t)lo * ncols * 4, dist_stage.p,
                                    (size_t)(hi - lo) * ncols * 4, cudaMemcpyDeviceToHost, st));
        if (pred && !pred_dev)
            WR_CUDA(cudaMemcpyAsync(pred + (size_t)lo * V, pred_stage.p, (size_t)(hi - lo) * V * 4,
                                    cudaMemcpyDeviceToHost, st));
        ++segments;
        total_tiles += ntiles;
    }
    WR_CUDA(cudaEventRecord(e1, st));
    BfTileStats hs{};
    WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    if (!o.async || !dist_dev || (pred && !pred_dev)) WR_CUDA(cudaStreamSynchronize(st));
    else WR_CUDA(cudaStreamSynchronize(st));  // stats/temporaries need the sync; async reserved
    float ms = 0.f;
    WR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats) {
        stats->rounds_max = hs.rounds_max;
        stats->relaxations = (int64_t)hs.relax;
        stats->segments = segments;
        stats->tiles = (int32_t)total_tiles;
        stats->ms = ms;
        stats->negcycle_source = -1;
        stats->kernel_launches = g_launches - g_launch0;
    }
    return WR_OK;
}

}  // namespace wr

extern "C" wr_status wr_bf_batch(const wr_graph *g, const int32_t *sources, int32_t S, const int32_t *targets,
                                 int32_t T, void *dist, int32_t *pred, const wr_bf_opts *opts,
                                 wr_bf_stats *stats) {
    return wr::guarded([&] { return wr::bf_batch_impl(g, sources, S, targets, T, dist, pred, opts, stats); });
}
