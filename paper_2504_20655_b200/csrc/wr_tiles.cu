// wr_tiles.cu - source-tile formation for the relaxation sweep (a3/a8).
//
// A tile's 32*SPL sources share one frontier: a vertex is re-relaxed for all
// of them whenever any of them improves it, so the work per tile grows with
// the spread of the sources' wavefronts. When the graph carries location
// coordinates (x, y and optionally the rack level z), the sources of a
// segment are ordered along a Morton (Z-order) curve before they are cut
// into tiles, so each tile is a compact box of nearby locations. Without
// coordinates the sorted vertex order is kept. The order is a stable sort
// (ties keep the sorted source order), done by a device LSD radix sort, and
// it only changes which sources share a tile - every result is per source
// and bit-identical either way (O2 fixpoint).
#include <algorithm>

#include <climits>
#include <thread>
#include <vector>
#include <cstdlib>
#include "wr_internal.cuh"

namespace wr {

__device__ __forceinline__ int bits_for(int range) {   // bits to hold [0, range]
    return range <= 0 ? 0 : 32 - __clz(range);
}

__global__ void morton_keys_kernel(const int *sources, int64_t lo, int n, const int *xy, const int *z, int xmin,
                                   int xmax, int ymin, int ymax, int zmin, int zmax, uint32_t *keys, int *idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = sources[lo + i];
    const uint32_t c[3] = {(uint32_t)(xy[2 * v] - xmin), (uint32_t)(xy[2 * v + 1] - ymin),
                           z ? (uint32_t)(z[v] - zmin) : 0u};
    const int nb[3] = {bits_for(xmax - xmin), bits_for(ymax - ymin), z ? bits_for(zmax - zmin) : 0};
    const int top = max(nb[0], max(nb[1], nb[2]));
    uint64_t key = 0;
    int total = 0;
    for (int b = top - 1; b >= 0; --b) {          // most significant level first
        for (int d = 0; d < 3; ++d) {
            if (b < nb[d]) {
                key = (key << 1) | ((c[d] >> b) & 1u);
                ++total;
            }
        }
    }
    keys[i] = total > 32 ? (uint32_t)(key >> (total - 32)) : (uint32_t)key;
    idx[i] = i;
}

// ------------------------------------------------ stable LSD radix sort --
constexpr int RS_ITEMS = 2048;

__global__ void __launch_bounds__(256) rs_hist_kernel(const uint32_t *keys, int n, int shift, int nblocks,
                                                      int *counts) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int b0 = blockIdx.x * RS_ITEMS, b1 = min(n, b0 + RS_ITEMS);
    for (int i = b0 + threadIdx.x; i < b1; i += 256) atomicAdd(&h[(keys[i] >> shift) & 255u], 1);
    __syncthreads();
    counts[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// One warp per block walks its items in order; __match_any_sync ranks equal
// digits inside each 32-item step, so the scatter is stable.
__global__ void __launch_bounds__(32) rs_scatter_kernel(const uint32_t *kin, const int *vin, uint32_t *kout,
                                                        int *vout, int n, int shift, int nblocks,
                                                        const int *offsets) {
    __shared__ int run[256];
    const int lane = threadIdx.x;
    for (int d = lane; d < 256; d += 32) run[d] = offsets[d * nblocks + blockIdx.x];
    __syncwarp();
    const int b0 = blockIdx.x * RS_ITEMS, b1 = min(n, b0 + RS_ITEMS);
    const unsigned lt = (1u << lane) - 1u;
    for (int base = b0; base < b1; base += 32) {
        const int i = base + lane;
        const bool valid = i < b1;
        const uint32_t k = valid ? kin[i] : 0u;
        const int d = valid ? (int)((k >> shift) & 255u) : 256 + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        const int pos = valid ? run[d] + rank : 0;
        __syncwarp();
        if (valid) {
            kout[pos] = k;
            vout[pos] = vin[i];
            if (rank == 0) run[d] += __popc(peers);
        }
        __syncwarp();
    }
}

static void radix_sort_pairs(uint32_t *keys, int *vals, uint32_t *ktmp, int *vtmp, int n, cudaStream_t st) {
    const int nblocks = (n + RS_ITEMS - 1) / RS_ITEMS;
    DBuf<int> counts((size_t)256 * nblocks);
    uint32_t *ka = keys, *kb = ktmp;
    int *va = vals, *vb = vtmp;
    for (int shift = 0; shift < 32; shift += 8) {
        rs_hist_kernel<<<nblocks, 256, 0, st>>>(ka, n, shift, nblocks, counts.p);
        count_launch();
        WR_LAUNCH_CHECK();
        scan_exclusive_i32(counts.p, counts.p, 256 * nblocks, st);
        rs_scatter_kernel<<<nblocks, 32, 0, st>>>(ka, va, kb, vb, n, shift, nblocks, counts.p);
        count_launch();
        WR_LAUNCH_CHECK();
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    // 4 passes: the result is back in (keys, vals)
    WR_CUDA(cudaStreamSynchronize(st));
}

// Tile t holds the sources perm[t*fill .. t*fill + fill) in its first fill
// slots; the remaining slots of the tsw-slot tile are empty (-1).
__global__ void tiles_from_perm_kernel(const int *sources, int64_t lo, const int *perm, int n, int fill, int tsw,
                                       int total, int *tile_src, int *slot_row, int *pos_of) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= total) return;
    const int t = p / tsw, k = p % tsw;
    const int q = t * fill + k;
    if (k < fill && q < n) {
        const int i = perm ? perm[q] : q;
        tile_src[p] = sources[lo + i];
        slot_row[p] = i;
        pos_of[i] = p;
    } else {
        tile_src[p] = -1;
        slot_row[p] = -1;
    }
}

// Recursive coordinate bisection of the sources into tiles (host): a node
// of k = ceil(n / tsw) tiles is split along the longest side of its
// bounding box (x, y at scale 2, rack level at scale 1: a level step is
// half an aisle step in the generators' weights) so that the left part
// holds exactly floor(k / 2) full tiles; leaves are single tiles, the only
// partial tile is the last leaf. Measured on C5: a Morton-curve cut makes
// some tiles straddle a curve jump (span 31-63 cells instead of 7), and a
// tile's sweep time follows its spatial spread (corr 0.69; 17 ms compact
// vs 40-52 ms straddling), not its rounds.
static void rcb(int *idx, int n, int tsw, const int *cx, const int *cy, const int *cz, int depth = 0) {
    if (n <= tsw) return;
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (int i = 0; i < n; ++i) {
        const int c[3] = {cx[idx[i]], cy[idx[i]], cz[idx[i]]};
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], c[a]);
            hi[a] = std::max(hi[a], c[a]);
        }
    }
    int axis = 0;
    for (int a = 1; a < 3; ++a)
        if (hi[a] - lo[a] > hi[axis] - lo[axis]) axis = a;
    const int *key = axis == 0 ? cx : axis == 1 ? cy : cz;
    const int k = (n + tsw - 1) / tsw;
    const int nl = (k / 2) * tsw;
    std::nth_element(idx, idx + nl, idx + n, [&](int a, int b) { return key[a] < key[b] || (key[a] == key[b] && a < b); });
    if (depth < 4 && n > 8192) {   // the two halves are independent: top levels on host threads
        std::thread left([=] { rcb(idx, nl, tsw, cx, cy, cz, depth + 1); });
        rcb(idx + nl, n - nl, tsw, cx, cy, cz, depth + 1);
        left.join();
    } else {
        rcb(idx, nl, tsw, cx, cy, cz, depth + 1);
        rcb(idx + nl, n - nl, tsw, cx, cy, cz, depth + 1);
    }
}

static bool rcb_perm(const wr_graph *g, const int *d_sources, int64_t lo, int n, int tsw, int *d_perm,
                     cudaStream_t st) {
    if (g->h_xy.empty()) {   // host copy of the coordinates, once per graph
        g->h_xy.resize((size_t)2 * g->V);
        WR_CUDA(cudaMemcpy(g->h_xy.data(), g->xy.p, 8 * (size_t)g->V, cudaMemcpyDeviceToHost));
        g->h_z.assign(g->V, 0);
        if (g->z.p) WR_CUDA(cudaMemcpy(g->h_z.data(), g->z.p, 4 * (size_t)g->V, cudaMemcpyDeviceToHost));
    }
    std::vector<int> src(n), cx(n), cy(n), cz(n), idx(n);
    WR_CUDA(cudaMemcpyAsync(src.data(), d_sources + lo, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i) {
        const int v = src[i];
        cx[i] = 2 * g->h_xy[2 * (size_t)v];
        cy[i] = 2 * g->h_xy[2 * (size_t)v + 1];
        cz[i] = g->h_z[v];
        idx[i] = i;
    }
    rcb(idx.data(), n, tsw, cx.data(), cy.data(), cz.data());
    WR_CUDA(cudaMemcpyAsync(d_perm, idx.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    WR_CUDA(cudaStreamSynchronize(st));   // idx lifetime
    return true;
}

// Tile count: by default ceil(n / tsw) full tiles. WR_TILE_BALANCE=1 spreads
// the sources over a whole number of waves instead (one tile per SM at a
// time; fill sources per tile). Measured on C5 packed: the sweep does not
// gain (a tile's time is latency-bound, nearly independent of its fill: 331
// full tiles 61 ms, 444 tiles of 191 sources 62 ms) and the pred pass, whose
// cost is per (tile, vertex) job, loses 20 % (32 -> 39.7 ms).
int balanced_tiles(int64_t n, int tsw, int64_t max_tiles, int &fill) {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        WR_CUDA(cudaGetDevice(&dev));
        WR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    static const bool off = getenv("WR_TILE_BALANCE") == nullptr;
    const int64_t base = (n + tsw - 1) / tsw;
    int64_t nt = base;
    if (!off) {
        const int64_t waves = (base + nsm - 1) / nsm;
        nt = std::max<int64_t>(base, std::min<int64_t>({waves * nsm, max_tiles, n}));
    }
    fill = (int)((n + nt - 1) / std::max<int64_t>(nt, 1));
    return (int)((n + fill - 1) / std::max(fill, 1));
}

int64_t tiles_to_allocate(int64_t sb, int tsw, int64_t extra_bytes, int64_t tile_bytes) {
    // extra tiles only serve the opt-in balancing; without it the buffer size
    // must not depend on the budget path (a repeated call then reuses the
    // cached block instead of growing the pool: 1.7 s for 34 GB)
    static const bool balance = getenv("WR_TILE_BALANCE") != nullptr;
    if (!balance) return sb / tsw;
    int nsm = 0, dev = 0;
    WR_CUDA(cudaGetDevice(&dev));
    WR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t base = sb / tsw;
    const int64_t extra = std::min<int64_t>(nsm - 1, std::max<int64_t>(0, extra_bytes / std::max<int64_t>(tile_bytes, 1)));
    return base + extra;
}

int make_tiles_ordered(const wr_graph *g, const int *d_sources, int64_t lo, int64_t hi, int tsw, int64_t max_tiles,
                       int *tile_src, int *slot_row, int *pos_of, cudaStream_t st) {
    const int n = (int)(hi - lo);
    if (n <= 0) return 0;
    int fill = tsw;
    const int ntiles = balanced_tiles(n, tsw, max_tiles, fill);
    const int total = ntiles * tsw;
    DBuf<int> perm;
    static const bool morton = getenv("WR_TILES_MORTON") != nullptr;
    if (g->xy.p && n > fill && !morton) {
        perm.alloc(n);
        rcb_perm(g, d_sources, lo, n, fill, perm.p, st);
    } else if (g->xy.p && n > fill) {
        DBuf<uint32_t> keys(n), ktmp(n);
        DBuf<int> vtmp(n);
        perm.alloc(n);
        morton_keys_kernel<<<(n + 255) / 256, 256, 0, st>>>(d_sources, lo, n, g->xy.p, g->z.p, g->bbox[0],
                                                            g->bbox[1], g->bbox[2], g->bbox[3], g->bbox[4],
                                                            g->bbox[5], keys.p, perm.p);
        count_launch();
        WR_LAUNCH_CHECK();
        radix_sort_pairs(keys.p, perm.p, ktmp.p, vtmp.p, n, st);
    }
    tiles_from_perm_kernel<<<(total + 255) / 256, 256, 0, st>>>(d_sources, lo, perm.p, n, fill, tsw, total,
                                                               tile_src, slot_row, pos_of);
    count_launch();
    WR_LAUNCH_CHECK();
    WR_CUDA(cudaStreamSynchronize(st));   // perm lifetime
    return ntiles;
}

}  // namespace wr
