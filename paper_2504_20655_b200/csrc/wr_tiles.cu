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

// Recursive coordinate bisection of the sources into tiles, on the device:
// a node of k = ceil(n / tsw) tiles is split along the longest side of its
// bounding box (x, y at scale 2, rack level at scale 1: a level step is
// half an aisle step in the generators' weights) so that the left part
// holds exactly floor(k / 2) full tiles; leaves are single tiles, the only
// partial tile is the last leaf. The tree's shape depends on n and tsw only,
// so the host lists every level's nodes up front and each level is one
// launch (one CTA per node: bounding box, radix select of the split key,
// stable partition) - no host round trip inside the step. Measured on C5: a
// Morton-curve cut makes some tiles straddle a curve jump (span 31-63 cells
// instead of 7), and a tile's sweep time follows its spatial spread (corr
// 0.69; 17 ms compact vs 40-52 ms straddling), not its rounds.
constexpr int RCB_NT = 1024;
constexpr uint32_t RCB_FULL = 0xffffffffu;
constexpr int RCB_BINS = 4096;   // 12-bit digits

// the sources' coordinates with their index, one 16-B element each, so every
// pass over a node is a coalesced read and the partition moves whole elements
__global__ void rcb_coords_kernel(const int *sources, int64_t lo, int n, const int *xy, const int *z, int4 *pts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = sources[lo + i];
    pts[i] = make_int4(xy[2 * v], xy[2 * v + 1], z ? z[v] : 0, i);
}

__global__ void rcb_perm_kernel(const int4 *pts, int n, int *perm) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) perm[i] = pts[i].w;
}

__device__ __forceinline__ int rcb_comp(const int4 &p, int axis) { return axis == 0 ? p.x : axis == 1 ? p.y : p.z; }

// exclusive block scan of one int per thread (RCB_NT threads); returns the total
__device__ int rcb_scan(int x, int &excl, int *sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(RCB_FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = sh[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(RCB_FULL, wi, o);
            if (lane >= o) wi += y;
        }
        sh[lane] = wi - w;
        if (lane == 31) sh[32] = wi;
    }
    __syncthreads();
    excl = sh[warp] + inc - x;
    const int total = sh[32];
    __syncthreads();
    return total;
}

// node = {start, count, nl}: the first nl positions of the node's range end
// up holding sources whose split key is <= every key on the right
__global__ void __launch_bounds__(RCB_NT) rcb_level_kernel(const int4 *nodes, int4 *pts, int4 *tmp) {
    __shared__ int hist[RCB_BINS];
    __shared__ int sh[40];
    __shared__ int s_red[6][32];
    __shared__ int s_wlt[RCB_NT / 32], s_weq[RCB_NT / 32];
    const int4 nd = nodes[blockIdx.x];
    const int s = nd.x, n = nd.y, nl = nd.z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int4 *pt = pts + s;
    // ---- bounding box
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += RCB_NT) {
        const int4 p = pt[i];
        const int c[3] = {p.x, p.y, p.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = min(mn[a], c[a]);
            mx[a] = max(mx[a], c[a]);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        mn[a] = __reduce_min_sync(RCB_FULL, mn[a]);
        mx[a] = __reduce_max_sync(RCB_FULL, mx[a]);
        if (lane == 0) { s_red[a][warp] = mn[a]; s_red[3 + a][warp] = mx[a]; }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = __reduce_min_sync(RCB_FULL, s_red[a][lane]);
            mx[a] = __reduce_max_sync(RCB_FULL, s_red[3 + a][lane]);
        }
        if (lane == 0) {
            const long long side[3] = {2LL * ((long long)mx[0] - mn[0]), 2LL * ((long long)mx[1] - mn[1]),
                                       (long long)mx[2] - mn[2]};
            int axis = 0;
            for (int a = 1; a < 3; ++a)
                if (side[a] > side[axis]) axis = a;
            sh[34] = axis;
            sh[35] = mn[axis];
            sh[36] = (int)((uint32_t)mx[axis] - (uint32_t)mn[axis]);   // < 2^32
        }
    }
    __syncthreads();
    const int axis = sh[34];
    const int klo = sh[35];
    const uint32_t range = (uint32_t)sh[36];
    // ---- radix select: P = the key of rank nl (0-based) in the node
    int bits = 0;
    while (bits < 32 && (range >> bits)) ++bits;
    uint32_t prefix = 0;   // the high bits of P found so far
    int rank = nl;         // rank of P among the keys that share the prefix
    for (int hi = bits; hi > 0;) {   // digit = key bits [shift, hi), bits >= hi fixed by prefix
        const int shift = max(0, hi - 12);
        const uint32_t dmask = (1u << (hi - shift)) - 1u;
        for (int b = threadIdx.x; b < RCB_BINS; b += RCB_NT) hist[b] = 0;
        __syncthreads();
#pragma unroll 4
        for (int i = threadIdx.x; i < n; i += RCB_NT) {
            const uint32_t k = (uint32_t)rcb_comp(pt[i], axis) - (uint32_t)klo;
            if (hi >= 32 || (k >> hi) == (prefix >> hi)) atomicAdd(&hist[(k >> shift) & dmask], 1);
        }
        __syncthreads();
        constexpr int PER = RCB_BINS / RCB_NT;
        int part = 0;
#pragma unroll
        for (int b = 0; b < PER; ++b) part += hist[threadIdx.x * PER + b];
        int before = 0;
        rcb_scan(part, before, sh);
        if (rank >= before && rank < before + part) {   // exactly one thread
            int r = rank - before, b = threadIdx.x * PER;
            while (r >= hist[b]) r -= hist[b++];
            sh[37] = b;
            sh[38] = r;
        }
        __syncthreads();
        prefix |= (uint32_t)sh[37] << shift;
        rank = sh[38];
        __syncthreads();
        hi = shift;
    }
    const uint32_t P = prefix;
    // ---- stable partition: keys < P, then (nl - #less) keys == P, left. Each
    // warp owns a contiguous chunk read 32 elements at a time (coalesced);
    // ballots rank the elements inside a group, a block scan the warps
    constexpr int NWP = RCB_NT / 32;
    const int wchunk = ((n + NWP - 1) / NWP + 31) & ~31;
    const int w0 = min(n, warp * wchunk), w1 = min(n, w0 + wchunk);
    const unsigned below = (1u << lane) - 1u;
    int lt = 0, eq = 0;
#pragma unroll 4
    for (int i0 = w0; i0 < w1; i0 += 32) {
        const int i = i0 + lane;
        const uint32_t k = i < w1 ? (uint32_t)rcb_comp(pt[i], axis) - (uint32_t)klo : 0xffffffffu;
        lt += __popc(__ballot_sync(RCB_FULL, i < w1 && k < P));
        eq += __popc(__ballot_sync(RCB_FULL, i < w1 && k == P));
    }
    if (lane == 0) { s_wlt[warp] = lt; s_weq[warp] = eq; }
    __syncthreads();
    int lt0 = 0, eq0 = 0, nlt = 0;
    for (int q = 0; q < NWP; ++q) {   // warps before this one, and the totals
        if (q < warp) { lt0 += s_wlt[q]; eq0 += s_weq[q]; }
        nlt += s_wlt[q];
    }
    const int quota = nl - nlt;
    for (int i0 = w0; i0 < w1; i0 += 32) {
        const int i = i0 + lane;
        const bool ok = i < w1;
        int4 p = make_int4(0, 0, 0, 0);
        uint32_t k = 0xffffffffu;
        if (ok) {
            p = pt[i];
            k = (uint32_t)rcb_comp(p, axis) - (uint32_t)klo;
        }
        const unsigned mlt = __ballot_sync(RCB_FULL, ok && k < P);
        const unsigned meq = __ballot_sync(RCB_FULL, ok && k == P);
        const int eq_rank = eq0 + __popc(meq & below);   // rank among the node's P keys
        const bool eq_left = (meq >> lane) & 1u && eq_rank < quota;
        if (ok) {
            int pos;
            if ((mlt >> lane) & 1u) {
                pos = lt0 + __popc(mlt & below);
            } else if (eq_left) {
                pos = nlt + eq_rank;
            } else {
                // right side: every element before this one (node order) that is
                // not left - (i - lefts before i)
                const int left_before = lt0 + __popc(mlt & below) + min(eq0 + __popc(meq & below), quota);
                pos = nl + (i - left_before);
            }
            tmp[s + pos] = p;
        }
        lt0 += __popc(mlt);
        eq0 += __popc(meq);
    }
    __syncthreads();
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += RCB_NT) pt[i] = tmp[s + i];
}

// the tree's levels: count of internal nodes per depth (host) ...
static void rcb_level_sizes(int n, int tsw, int depth, std::vector<int> &cnt) {
    if (n <= tsw) return;
    const int k = (n + tsw - 1) / tsw, nl = (k / 2) * tsw;
    if ((int)cnt.size() <= depth) cnt.resize(depth + 1, 0);
    ++cnt[depth];
    rcb_level_sizes(nl, tsw, depth + 1, cnt);
    rcb_level_sizes(n - nl, tsw, depth + 1, cnt);
}

// ... and the same walk on the device writes the nodes (no host-to-device copy)
struct RcbLevels {
    int off[32];
};
__global__ void rcb_nodes_kernel(int n, int tsw, RcbLevels lv, int4 *nodes) {
    int cur[32];
    for (int d = 0; d < 32; ++d) cur[d] = lv.off[d];
    int st_s[64], st_n[64], st_d[64], top = 0;
    st_s[0] = 0; st_n[0] = n; st_d[0] = 0; top = 1;
    while (top > 0) {
        --top;
        const int s = st_s[top], m = st_n[top], d = st_d[top];
        if (m <= tsw) continue;
        const int k = (m + tsw - 1) / tsw, nl = (k / 2) * tsw;
        nodes[cur[d]++] = make_int4(s, m, nl, 0);
        st_s[top] = s + nl; st_n[top] = m - nl; st_d[top] = d + 1; ++top;
        st_s[top] = s; st_n[top] = nl; st_d[top] = d + 1; ++top;
    }
}

static void rcb_perm(const wr_graph *g, const int *d_sources, int64_t lo, int n, int tsw, int *d_perm,
                     cudaStream_t st) {
    std::vector<int> cnt;
    rcb_level_sizes(n, tsw, 0, cnt);
    if (cnt.size() > 32) WR_THROW(WR_EINTERNAL, "rcb: tree too deep");
    RcbLevels lv{};
    int total = 0;
    for (size_t L = 0; L < cnt.size(); ++L) {
        lv.off[L] = total;
        total += cnt[L];
    }
    DBuf<int4> pts(n), tmp(n);
    DBuf<int4> nodes(std::max(total, 1));
    rcb_nodes_kernel<<<1, 1, 0, st>>>(n, tsw, lv, nodes.p);
    count_launch();
    WR_LAUNCH_CHECK();
    rcb_coords_kernel<<<(n + 255) / 256, 256, 0, st>>>(d_sources, lo, n, g->xy.p, g->z.p, pts.p);
    count_launch();
    WR_LAUNCH_CHECK();
    for (size_t L = 0; L < cnt.size(); ++L) {
        rcb_level_kernel<<<cnt[L], RCB_NT, 0, st>>>(nodes.p + lv.off[L], pts.p, tmp.p);
        count_launch();
        WR_LAUNCH_CHECK();
    }
    rcb_perm_kernel<<<(n + 255) / 256, 256, 0, st>>>(pts.p, n, d_perm);
    count_launch();
    WR_LAUNCH_CHECK();
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
    return ntiles;   // temporaries go back to the stream-ordered pool
}

}  // namespace wr
