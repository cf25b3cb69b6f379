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

__global__ void tiles_from_perm_kernel(const int *sources, int64_t lo, const int *perm, int n, int total,
                                       int *tile_src, int *slot_row, int *pos_of) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= total) return;
    if (p < n) {
        const int i = perm ? perm[p] : p;
        tile_src[p] = sources[lo + i];
        slot_row[p] = i;
        pos_of[i] = p;
    } else {
        tile_src[p] = -1;
        slot_row[p] = -1;
    }
}

void make_tiles_ordered(const wr_graph *g, const int *d_sources, int64_t lo, int64_t hi, int tsw, int *tile_src,
                        int *slot_row, int *pos_of, cudaStream_t st) {
    const int n = (int)(hi - lo);
    const int total = (int)(((int64_t)n + tsw - 1) / tsw * tsw);
    if (total == 0) return;
    DBuf<int> perm;
    if (g->xy.p && n > tsw) {
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
    tiles_from_perm_kernel<<<(total + 255) / 256, 256, 0, st>>>(d_sources, lo, perm.p, n, total, tile_src,
                                                               slot_row, pos_of);
    count_launch();
    WR_LAUNCH_CHECK();
    WR_CUDA(cudaStreamSynchronize(st));   // perm lifetime
}

}  // namespace wr
