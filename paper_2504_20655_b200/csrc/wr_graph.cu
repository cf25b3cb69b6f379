// wr_graph.cu - a1 graph ingest (P721 §4.7: edge list u, v, w; S358-361),
// device scans, error plumbing and small ABI helpers.
//
// The ingest runs on the device: validation, degree histograms, exclusive
// scans, scatter into CSC (in-arcs) / CSR (out-arcs), and a per-vertex sort
// of the in-arcs by (tail, weight bits) so the layout is deterministic.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "wr_internal.cuh"

namespace wr {

static thread_local std::string g_err;
thread_local int64_t g_launches = 0;
thread_local cudaStream_t g_stream = 0;

// ----------------------------------------------------------- memory pool --
static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64] = {};

static cudaMemPool_t pool_for(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= 64) WR_THROW(WR_EINVAL, "device ordinal out of range");
    if (!g_pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        WR_CUDA(cudaMemPoolCreate(&g_pools[dev], &props));
        uint64_t thr = UINT64_MAX;
        WR_CUDA(cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
    }
    return g_pools[dev];
}

// Block cache in front of the pool: a freed block is kept (not returned to
// the pool) and handed back to the next request of a fitting size on the
// same stream - stream order makes the reuse safe - so a repeated call makes
// no allocation driver calls at all. Those calls were measured to stall the
// host for up to ~40 ms while another process (nvidia-smi sampling) held
// the driver. Cached blocks count as idle memory (pool_idle_bytes) and are
// released on OOM and by wr_release_cached.
struct CachedBlock {
    void *p;
    size_t bytes;
    cudaStream_t s;
    int dev;
};
static std::mutex g_cache_mu;
static std::vector<CachedBlock> g_cache;
static std::vector<std::pair<void *, size_t>> g_live;   // outstanding blocks and their sizes
constexpr size_t CACHE_MAX_BLOCKS = 256;

static void cache_release(int dev) {   // hand every cached block of dev back to the pool
    std::vector<CachedBlock> out;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (size_t i = 0; i < g_cache.size();) {
            if (g_cache[i].dev == dev) {
                out.push_back(g_cache[i]);
                g_cache[i] = g_cache.back();
                g_cache.pop_back();
            } else {
                ++i;
            }
        }
    }
    for (auto &b : out) cudaFreeAsync(b.p, b.s);
}

void *pool_alloc(size_t bytes, cudaStream_t s) {
    int dev = 0;
    WR_CUDA(cudaGetDevice(&dev));
    if (bytes == 0) bytes = 1;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        int best = -1;
        for (int i = 0; i < (int)g_cache.size(); ++i) {
            const CachedBlock &b = g_cache[i];
            // fits: at least the request, at most 1/8 (or 1 MB) larger
            if (b.dev == dev && b.s == s && b.bytes >= bytes && b.bytes - bytes <= std::max<size_t>(bytes / 8, 1 << 20) &&
                (best < 0 || b.bytes < g_cache[best].bytes))
                best = i;
        }
        if (best >= 0) {
            CachedBlock b = g_cache[best];
            g_cache[best] = g_cache.back();
            g_cache.pop_back();
            g_live.emplace_back(b.p, b.bytes);
            return b.p;
        }
    }
    void *p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool_for(dev), s);
    if (e == cudaErrorMemoryAllocation) {   // give cached and idle pool memory back and retry once
        cudaGetLastError();
        cache_release(dev);
        WR_CUDA(cudaDeviceSynchronize());
        WR_CUDA(cudaMemPoolTrimTo(pool_for(dev), 0));
        e = cudaMallocFromPoolAsync(&p, bytes, pool_for(dev), s);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("device allocation of ") + std::to_string(bytes) + " bytes: " + cudaGetErrorString(e));
        throw CudaError{e == cudaErrorMemoryAllocation ? WR_ENOMEM : WR_ECUDA};
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_live.emplace_back(p, bytes);
    return p;
}

void pool_free(void *p, cudaStream_t s) {
    if (!p) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeAsync(p, s);
        return;
    }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t bytes = 0;
    for (size_t i = 0; i < g_live.size(); ++i)
        if (g_live[i].first == p) {
            bytes = g_live[i].second;
            g_live[i] = g_live.back();
            g_live.pop_back();
            break;
        }
    if (bytes == 0 || g_cache.size() >= CACHE_MAX_BLOCKS) {
        cudaFreeAsync(p, s);
        return;
    }
    g_cache.push_back(CachedBlock{p, bytes, s, dev});
}

size_t pool_idle_bytes(int dev) {
    cudaMemPool_t pool = pool_for(dev);
    uint64_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    size_t cached = 0;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto &b : g_cache)
            if (b.dev == dev) cached += b.bytes;
    }
    return (reserved > used ? (size_t)(reserved - used) : 0) + cached;
}

NvtxRange::NvtxRange(const char *name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

void set_error(const std::string &msg) { g_err = msg; }
wr_status fail(wr_status code, const std::string &msg) {
    g_err = msg;
    return code;
}

bool is_device_ptr(const void *ptr) {
    if (!ptr) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int64_t factorial64(int n) {
    int64_t f = 1;
    for (int k = 2; k <= n; ++k) f *= k;
    return f;
}

// ------------------------------------------------------------------ scans --
constexpr int SCAN_T = 512;
constexpr int SCAN_PER = 4;
constexpr int SCAN_TILE = SCAN_T * SCAN_PER;

template <class T>
__global__ void __launch_bounds__(SCAN_T) scan_tiles_kernel(const T *in, T *out, T *block_sums, int64_t n) {
    __shared__ T warp_tot[SCAN_T / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_PER;
    T v[SCAN_PER];
    T run = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; ++k) {
        v[k] = (base + k < n) ? in[base + k] : T(0);
        T t = v[k];
        v[k] = run;           // exclusive within the thread
        run += t;
    }
    // exclusive scan of thread totals across the block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T x = (lane < SCAN_T / 32) ? warp_tot[lane] : T(0);
        T xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, xi, d);
            if (lane >= d) xi += y;
        }
        if (lane < SCAN_T / 32) warp_tot[lane] = xi - x;  // exclusive warp offsets
        if (lane == SCAN_T / 32 - 1 && block_sums) block_sums[blockIdx.x] = xi;
    }
    __syncthreads();
    const T off = warp_tot[warp] + (incl - run);
#pragma unroll
    for (int k = 0; k < SCAN_PER; ++k)
        if (base + k < n) out[base + k] = v[k] + off;
}

template <class T>
__global__ void scan_add_kernel(T *out, const T *block_off, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += block_off[i / SCAN_TILE];
}

template <class T>
static void scan_exclusive(const T *in, T *out, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (nb == 1) {
        scan_tiles_kernel<T><<<1, SCAN_T, 0, st>>>(in, out, nullptr, n);
        count_launch();
        WR_LAUNCH_CHECK();
        return;
    }
    DBuf<T> sums(nb);
    scan_tiles_kernel<T><<<(unsigned)nb, SCAN_T, 0, st>>>(in, out, sums.p, n);
    count_launch();
    WR_LAUNCH_CHECK();
    scan_exclusive<T>(sums.p, sums.p, nb, st);
    scan_add_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, sums.p, n);
    count_launch();
    WR_LAUNCH_CHECK();
    WR_CUDA(cudaStreamSynchronize(st));  // sums is freed on return
}

void scan_exclusive_i64(const int64_t *in, int64_t *out, int64_t n, cudaStream_t st) {
    scan_exclusive<int64_t>(in, out, n, st);
}
void scan_exclusive_i32(const int *in, int *out, int n, cudaStream_t st) {
    scan_exclusive<int>(in, out, n, st);
}

// ----------------------------------------------------------- ingest kernels --
enum : int { BAD_INDEX = 1, BAD_WEIGHT = 2, BAD_XY = 4 };

__global__ void csr_to_src_kernel(const int64_t *row_ptr, int V, int *src) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= V) return;
    for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) src[k] = u;
}

__global__ void validate_kernel(const int *src, const int *dst, uint32_t *w, int64_t E, int V, int wtype,
                                int *flags, unsigned *max_abs, int *has_neg, int *has_zero, int64_t *in_deg,
                                int64_t *out_deg) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int u = src[e], v = dst[e];
    if (u < 0 || u >= V || v < 0 || v >= V) {
        atomicOr(flags, BAD_INDEX);
        return;
    }
    uint32_t bits = w[e];
    if (wtype == WR_F32) {
        const float x = __uint_as_float(bits);
        if (!(x >= 0.0f) || isinf(x)) atomicOr(flags, BAD_WEIGHT);  // NaN, -x, inf
        if (bits == 0x80000000u) w[e] = 0u;                            // -0.0 -> +0.0
        else if (x >= 0.0f && !isinf(x)) atomicMax(max_abs, bits);     // fp32 >= 0: bit order = value order
    } else {
        const int x = (int)bits;
        if (x < 0) atomicOr(has_neg, 1);
        if (x == 0) atomicOr(has_zero, 1);
        const unsigned a = x < 0 ? (unsigned)(-(int64_t)x) : (unsigned)x;
        atomicMax(max_abs, a);
    }
    atomicAdd((unsigned long long *)&in_deg[v], 1ull);
    atomicAdd((unsigned long long *)&out_deg[u], 1ull);
}

__global__ void max_deg_kernel(const int64_t *deg, int V, unsigned long long *mx) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V) atomicMax(mx, (unsigned long long)deg[v]);
}

__global__ void validate_xy_kernel(const int *xy, int V, int *flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * V) return;
    const int x = xy[i];
    if (x <= -(1 << 20) || x >= (1 << 20)) atomicOr(flags, BAD_XY);
}

// bbox = {xmin, xmax, ymin, ymax, zmin, zmax}; also validates |z| < 2^20.
__global__ void bbox_kernel(const int *xy, const int *z, int V, int *bbox, int *flags) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    atomicMin(&bbox[0], xy[2 * v]);
    atomicMax(&bbox[1], xy[2 * v]);
    atomicMin(&bbox[2], xy[2 * v + 1]);
    atomicMax(&bbox[3], xy[2 * v + 1]);
    if (z) {
        const int zz = z[v];
        if (zz <= -(1 << 20) || zz >= (1 << 20)) atomicOr(flags, BAD_XY);
        atomicMin(&bbox[4], zz);
        atomicMax(&bbox[5], zz);
    }
}

__global__ void narrow_kernel(const int64_t *a, int *b, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (int)a[i];
}

__global__ void scatter_kernel(const int *src, const int *dst, const uint32_t *w, int64_t E,
                               int *in_cur, int *out_cur, int *in_src, uint32_t *in_w, int *out_dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int u = src[e], v = dst[e];
    const int pi = atomicAdd(&in_cur[v], 1);
    in_src[pi] = u;
    in_w[pi] = w[e];
    const int po = atomicAdd(&out_cur[u], 1);
    out_dst[po] = v;
}

// Deterministic order: in-arcs of v sorted by (tail, weight bits); out-arcs
// of u sorted by head. Insertion sort per vertex (warehouse degrees <= ~10).
__global__ void pack_arcs_kernel(const int *in_src, const uint32_t *in_w, int2 *in_arc, int64_t E) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < E) in_arc[i] = make_int2(in_src[i], (int)in_w[i]);
}

__global__ void sort_adj_kernel(const int *in_ptr, int *in_src, uint32_t *in_w, const int *out_ptr,
                                int *out_dst, int V) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    for (int a = in_ptr[v] + 1; a < in_ptr[v + 1]; ++a) {
        const int u = in_src[a];
        const uint32_t x = in_w[a];
        int b = a - 1;
        while (b >= in_ptr[v] && (in_src[b] > u || (in_src[b] == u && in_w[b] > x))) {
            in_src[b + 1] = in_src[b];
            in_w[b + 1] = in_w[b];
            --b;
        }
        in_src[b + 1] = u;
        in_w[b + 1] = x;
    }
    for (int a = out_ptr[v] + 1; a < out_ptr[v + 1]; ++a) {
        const int x = out_dst[a];
        int b = a - 1;
        while (b >= out_ptr[v] && out_dst[b] > x) {
            out_dst[b + 1] = out_dst[b];
            --b;
        }
        out_dst[b + 1] = x;
    }
}

static unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static wr_status graph_load_impl(const wr_graph_desc *d, wr_graph **out) {
    if (!d || !out) return fail(WR_EINVAL, "wr_graph_load: null argument");
    *out = nullptr;
    if (d->V < 1 || d->V > (1 << 30)) return fail(WR_EINVAL, "wr_graph_load: V out of range");
    if (d->E < 0 || d->E >= ((int64_t)1 << 31)) return fail(WR_EINVAL, "wr_graph_load: E out of range");
    if (d->wtype != WR_I32 && d->wtype != WR_F32) return fail(WR_EINVAL, "wr_graph_load: wtype");
    if (d->format != WR_COO && d->format != WR_CSR) return fail(WR_EINVAL, "wr_graph_load: format");
    if (d->E > 0 && !d->w) return fail(WR_EINVAL, "wr_graph_load: weights missing");
    if (d->E > 0 && d->format == WR_COO && (!d->src || !d->dst))
        return fail(WR_EINVAL, "wr_graph_load: COO arrays missing");
    if (d->format == WR_CSR && (!d->row_ptr || (d->E > 0 && !d->col)))
        return fail(WR_EINVAL, "wr_graph_load: CSR arrays missing");
    int ndev = 0;
    WR_CUDA(cudaGetDeviceCount(&ndev));
    if (d->device < 0 || d->device >= ndev) return fail(WR_EINVAL, "wr_graph_load: bad device");
    WR_CUDA(cudaSetDevice(d->device));

    const int V = d->V;
    const int64_t E = d->E;
    cudaStream_t st = 0;
    auto g = std::make_unique<wr_graph>();
    g->device = d->device;
    g->V = V;
    g->E = E;
    g->wtype = d->wtype;

    DBuf<int> src(E), dst;
    if (d->format == WR_COO) {
        if (E) WR_CUDA(cudaMemcpyAsync(src.p, d->src, E * 4, cudaMemcpyDefault, st));
        dst = to_device<int>(d->dst, E, st);
    } else {
        std::vector<int64_t> rp(V + 1);
        WR_CUDA(cudaMemcpy(rp.data(), d->row_ptr, (V + 1) * 8, cudaMemcpyDefault));
        if (rp[0] != 0 || rp[V] != E) return fail(WR_EINVAL, "wr_graph_load: row_ptr must span [0, E]");
        for (int u = 0; u < V; ++u)
            if (rp[u + 1] < rp[u]) return fail(WR_EINVAL, "wr_graph_load: row_ptr not monotone");
        DBuf<int64_t> drp = to_device<int64_t>(rp.data(), V + 1, st);
        csr_to_src_kernel<<<grid_for(V, 256), 256, 0, st>>>(drp.p, V, src.p);
        count_launch();
        WR_LAUNCH_CHECK();
        dst = to_device<int>(d->col, E, st);
        WR_CUDA(cudaStreamSynchronize(st));
    }
    DBuf<uint32_t> w = to_device<uint32_t>((const uint32_t *)d->w, E, st);

    DBuf<int> flags(4);          // [0] flags, [1] max_abs, [2] has_neg, [3] has_zero (int)
    DBuf<int64_t> in_deg(V + 1), out_deg(V + 1);
    WR_CUDA(cudaMemsetAsync(flags.p, 0, 16, st));
    WR_CUDA(cudaMemsetAsync(in_deg.p, 0, (V + 1) * 8, st));
    WR_CUDA(cudaMemsetAsync(out_deg.p, 0, (V + 1) * 8, st));
    if (E) {
        validate_kernel<<<grid_for(E, 256), 256, 0, st>>>(src.p, dst.p, w.p, E, V, d->wtype, flags.p,
                                                         (unsigned *)(flags.p + 1), flags.p + 2, flags.p + 3,
                                                         in_deg.p, out_deg.p);
        count_launch();
        WR_LAUNCH_CHECK();
    }
    DBuf<int> bbox(6);
    if (d->xy) {
        g->xy = to_device<int>(d->xy, (size_t)V * 2, st);
        validate_xy_kernel<<<grid_for(2 * (int64_t)V, 256), 256, 0, st>>>(g->xy.p, V, flags.p);
        count_launch();
        WR_LAUNCH_CHECK();
        if (d->z) g->z = to_device<int>(d->z, (size_t)V, st);
        const int init[6] = {INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN, 0, 0};
        WR_CUDA(cudaMemcpyAsync(bbox.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
        if (d->z) {
            const int zi[2] = {INT32_MAX, INT32_MIN};
            WR_CUDA(cudaMemcpyAsync(bbox.p + 4, zi, sizeof(zi), cudaMemcpyHostToDevice, st));
        }
        bbox_kernel<<<grid_for(V, 256), 256, 0, st>>>(g->xy.p, g->z.p, V, bbox.p, flags.p);
        count_launch();
        WR_LAUNCH_CHECK();
        WR_CUDA(cudaMemcpyAsync(g->bbox, bbox.p, sizeof(g->bbox), cudaMemcpyDeviceToHost, st));
    }
    DBuf<unsigned long long> maxdeg(1);
    WR_CUDA(cudaMemsetAsync(maxdeg.p, 0, 8, st));
    max_deg_kernel<<<grid_for(V, 256), 256, 0, st>>>(in_deg.p, V, maxdeg.p);
    count_launch();
    WR_LAUNCH_CHECK();
    unsigned long long hmaxdeg = 0;
    WR_CUDA(cudaMemcpyAsync(&hmaxdeg, maxdeg.p, 8, cudaMemcpyDeviceToHost, st));
    int hf[4];
    WR_CUDA(cudaMemcpyAsync(hf, flags.p, 16, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    if (hf[0] & BAD_INDEX) return fail(WR_EINVAL, "wr_graph_load: arc endpoint outside [0, V)");
    if (hf[0] & BAD_WEIGHT) return fail(WR_EINVAL, "wr_graph_load: fp32 weight NaN, infinite or negative");
    if (hf[0] & BAD_XY) return fail(WR_EINVAL, "wr_graph_load: |xy| >= 2^20");
    g->has_negative = hf[2];
    g->has_zero = hf[3];
    g->max_abs_w = d->wtype == WR_I32 ? hf[1] : 0;
    if (d->wtype == WR_F32) memcpy(&g->max_w_f, &hf[1], 4);
    g->max_in_deg = (int64_t)hmaxdeg;
    if (d->wtype == WR_I32 && (int64_t)(V - 1) * (int64_t)(uint32_t)hf[1] >= (int64_t)INT32_MAX)
        return fail(WR_EOVERFLOW, "wr_graph_load: (V-1)*max|w| >= INT32_MAX (reading A7)");

    // offsets: exclusive scans of the degrees
    scan_exclusive_i64(in_deg.p, in_deg.p, V + 1, st);
    scan_exclusive_i64(out_deg.p, out_deg.p, V + 1, st);
    g->in_ptr.alloc(V + 1);
    g->out_ptr.alloc(V + 1);
    narrow_kernel<<<grid_for(V + 1, 256), 256, 0, st>>>(in_deg.p, g->in_ptr.p, V + 1);
    narrow_kernel<<<grid_for(V + 1, 256), 256, 0, st>>>(out_deg.p, g->out_ptr.p, V + 1);
    count_launch();
    count_launch();
    WR_LAUNCH_CHECK();
    g->in_src.alloc(std::max<int64_t>(E, 1));
    g->in_w.alloc(std::max<int64_t>(E, 1));
    g->out_dst.alloc(std::max<int64_t>(E, 1));
    if (E) {
        DBuf<int> in_cur(V + 1), out_cur(V + 1);
        WR_CUDA(cudaMemcpyAsync(in_cur.p, g->in_ptr.p, (V + 1) * 4, cudaMemcpyDeviceToDevice, st));
        WR_CUDA(cudaMemcpyAsync(out_cur.p, g->out_ptr.p, (V + 1) * 4, cudaMemcpyDeviceToDevice, st));
        scatter_kernel<<<grid_for(E, 256), 256, 0, st>>>(src.p, dst.p, w.p, E, in_cur.p, out_cur.p,
                                                        g->in_src.p, g->in_w.p, g->out_dst.p);
        count_launch();
        WR_LAUNCH_CHECK();
        sort_adj_kernel<<<grid_for(V, 128), 128, 0, st>>>(g->in_ptr.p, g->in_src.p, g->in_w.p,
                                                         g->out_ptr.p, g->out_dst.p, V);
        count_launch();
        WR_LAUNCH_CHECK();
        g->in_arc.alloc(E);
        pack_arcs_kernel<<<grid_for(E, 256), 256, 0, st>>>(g->in_src.p, g->in_w.p, g->in_arc.p, E);
        count_launch();
        WR_LAUNCH_CHECK();
        WR_CUDA(cudaStreamSynchronize(st));
    }
    WR_CUDA(cudaStreamSynchronize(st));
    *out = g.release();
    return WR_OK;
}

}  // namespace wr

extern "C" {

const char *wr_last_error(void) { return wr::g_err.c_str(); }
int32_t wr_version(void) { return 1; }

wr_status wr_release_cached(int32_t device) {
    return wr::guarded([&] {
        WR_CUDA(cudaSetDevice(device));
        WR_CUDA(cudaDeviceSynchronize());
        wr::cache_release(device);
        WR_CUDA(cudaDeviceSynchronize());
        WR_CUDA(cudaMemPoolTrimTo(wr::pool_for(device), 0));
        return WR_OK;
    });
}

wr_status wr_graph_load(const wr_graph_desc *desc, wr_graph **out) {
    return wr::guarded([&] {
        wr::NvtxRange nv("wr_graph_load");
        return wr::graph_load_impl(desc, out);
    });
}

wr_status wr_graph_free(wr_graph *g) {
    if (!g) return WR_OK;
    return wr::guarded([&] {
        WR_CUDA(cudaSetDevice(g->device));
        delete g;
        return WR_OK;
    });
}

wr_status wr_graph_info(const wr_graph *g, wr_graph_info_t *info) {
    if (!g || !info) return wr::fail(WR_EINVAL, "wr_graph_info: null argument");
    info->V = g->V;
    info->E = g->E;
    info->wtype = g->wtype;
    info->has_negative = g->has_negative;
    info->has_xy = g->xy.p != nullptr;
    info->device = g->device;
    info->device_bytes = (int64_t)(g->in_ptr.bytes() + g->in_src.bytes() + g->in_w.bytes() + g->in_arc.bytes() +
                                   g->out_ptr.bytes() + g->out_dst.bytes() + g->xy.bytes());
    info->max_abs_weight = g->wtype == WR_I32 ? g->max_abs_w : 0;
    return WR_OK;
}

void wr_shard_range(int64_t n, int32_t rank, int32_t world, int64_t *lo, int64_t *hi) {
    if (world < 1) world = 1;
    if (rank < 0) rank = 0;
    if (rank >= world) rank = world - 1;
    *lo = n * rank / world;
    *hi = n * (rank + 1) / world;
}

wr_status wr_route_count_reduction(int32_t m, const int32_t *n_j, uint64_t *reduced, uint64_t *brute) {
    // Theorem 3.1 (P326-329 §3): m! 2^(m-1) + (1/2) sum n_j!; brute n!/2.
    if (m < 1 || m > 20 || !n_j || !reduced || !brute) return wr::fail(WR_EINVAL, "wr_route_count_reduction");
    int64_t n = 0;
    uint64_t half = 0;
    for (int j = 0; j < m; ++j) {
        if (n_j[j] < 1 || n_j[j] > 20) return wr::fail(WR_EINVAL, "wr_route_count_reduction: n_j");
        n += n_j[j];
        half += (uint64_t)wr::factorial64(n_j[j]);
    }
    if (n > 20) return wr::fail(WR_ETOOLARGE, "wr_route_count_reduction: n > 20");
    *reduced = (uint64_t)wr::factorial64(m) * (1ull << (m - 1)) + half / 2;
    *brute = (uint64_t)wr::factorial64((int)n) / 2;
    return WR_OK;
}

}  // extern "C"
