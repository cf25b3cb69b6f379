// wr_route.cu - route evaluation over pick-node sequences (a5-a7), the
// Theorem 3.1 segmented route, the O8 segment plan, and the orders
// pipeline (a2..a9 phases) behind wr_route_orders.
//
// Paper: exhaustive evaluation of all n! orderings, one thread per
// permutation with an (n-1)-transition inner loop (P658 §4.6), memory errors
// above N = 2,903,040 permutations; clusters stitched through two boundary
// nodes each (Thm 3.1, P324-337 §3).
// Here: the n! sequences of a (sub)problem are the leaves of the permutation
// prefix trie (reading A18); a lane owns a lexicographic prefix and walks its
// subtree depth-first, so every internal trie node costs ONE add shared by
// all leaves below it (~e adds per leaf instead of n-1) and the left-to-right
// association of O4 is kept exactly. Work items are rank ranges of at most
// opts.chunk permutations (O6); per-lane minima are packed (cost key << 32 |
// rank) and reduced with integer min: ties resolve to the smallest rank =
// lexicographically smallest sequence (O5). Nothing is materialised per
// permutation, so the paper's memory limit disappears; the chunk only bounds
// the work of one warp.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include <cooperative_groups.h>

#include "wr_internal.cuh"

namespace wr {

constexpr int MS = WR_MAX_STOPS;      // 16
constexpr int DSTRIDE = MS * MS;      // D entries per order (row-major 16 x 16)
// exact routes of SHK_MIN..SHK_MAX stops go to the warp Held-Karp kernel
#ifndef SHK_MIN
#define SHK_MIN 8
#endif
#ifndef SHK_MAX
#define SHK_MAX 8
#endif

// ------------------------------------------------------------ cost ops --
// Route costs: int32 exact (with negatives possible when D < 0), fp32 RN.
// key(): order-preserving map to uint32 (fp32 costs are >= 0 or +inf).
struct CostI32 {
    static constexpr uint32_t INF = 0x7fffffffu;
    __device__ __forceinline__ static uint32_t add(uint32_t a, uint32_t b) { return (uint32_t)((int)a + (int)b); }
    __device__ __forceinline__ static uint32_t key(uint32_t c) { return c ^ 0x80000000u; }
    __device__ __forceinline__ static uint32_t unkey(uint32_t k) { return k ^ 0x80000000u; }
};
struct CostF32 {
    static constexpr uint32_t INF = 0x7f800000u;
    __device__ __forceinline__ static uint32_t add(uint32_t a, uint32_t b) {
        return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(b)));
    }
    __device__ __forceinline__ static uint32_t key(uint32_t c) { return c; }
    __device__ __forceinline__ static uint32_t unkey(uint32_t k) { return k; }
};

__host__ __device__ inline int64_t fact(int n) {
    int64_t f = 1;
    for (int k = 2; k <= n; ++k) f *= k;
    return f;
}

// p(n): prefix depth; a lane walks subtrees of (n-p)! leaves. Chosen to
// minimise the warp's cost ceil(P/32) * (decode + leaves * ~12 instr),
// P = n!/(n-p)! prefixes, with subtrees of at most 7! leaves (template depth).
__host__ __device__ inline int prefix_depth(int n) {
    if (n <= 1) return 0;
    int best_p = n - 1;
    int64_t best_c = -1;
    for (int p = (n - 7 > 1 ? n - 7 : 1); p <= n - 1; ++p) {
        const int64_t P = fact(n) / fact(n - p);
        const int64_t c = ((P + 31) / 32) * (40 + 12 * fact(n - p));
        if (best_c < 0 || c < best_c) {
            best_c = c;
            best_p = p;
        }
    }
    return best_p;
}
int route_prefix_depth(int n) { return prefix_depth(n); }

__constant__ uint32_t c_fact[13] = {1u, 1u, 2u, 6u, 24u, 120u, 720u, 5040u, 40320u, 362880u, 3628800u,
                                    39916800u, 479001600u};

// Lehmer decode of rank r over n elements into nibble-packed positions.
__device__ inline uint64_t unrank_nib(int64_t r, int n) {
    uint32_t unused = (1u << n) - 1u;
    uint64_t out = 0;
    for (int k = 0; k < n; ++k) {
        const int64_t f = fact(n - 1 - k);
        int q = (int)(r / f);
        r %= f;
        uint32_t m = unused;
        for (int t = 0; t < q; ++t) m &= m - 1;
        const int x = __ffs(m) - 1;
        unused &= ~(1u << x);
        out |= (uint64_t)x << (4 * k);
    }
    return out;
}

__device__ inline int nib(uint64_t v, int k) { return (int)((v >> (4 * k)) & 0xf); }

// ---------------------------------------------------------- trie walk --
// Leaves are visited in lexicographic order, so within a lane ranks only
// grow and a strict "<" on the cost key keeps the smallest rank (O5).
struct Best {
    uint32_t key;
    uint32_t rank;
};

template <class C>
__device__ __forceinline__ void leaf(uint32_t cost, Best &best, uint32_t &rank) {
    const uint32_t k = C::key(cost);
    if (k < best.key) {
        best.key = k;
        best.rank = rank;
    }
    ++rank;
}

// Ds rows have stride ns. CL (closed tour, NEXT-4): the depot is local
// index ns - 1; the walk starts there (prev = ns - 1, cost 0) and every
// leaf adds the return leg to it.
// The matrix is replicated per lane (element e of lane l at word e * 32 + l,
// Ds already offset by the lane): the 32 lanes of a warp walk different
// subtrees and read different elements, which in a single copy collide in
// shared-memory banks; one copy per lane puts every lane in its own bank.
#define DSL(e) Ds[(e) << SH]
template <class C, bool CL, int SH>
__device__ __forceinline__ uint32_t ret_leg(const uint32_t *Ds, int ns, int last, uint32_t cost) {
    if constexpr (CL) return C::add(cost, DSL(last * ns + ns - 1));
    return cost;
}

// PR (branch and bound, legs known >= 0 so prefix costs never decrease): a
// child whose prefix key already exceeds min(B, the lane's best key) holds
// no leaf that could win (ties are kept: the test is strict), so its
// (L-1)! leaves are skipped and only counted in the rank.
// The bound adds the legs still to come: every unvisited stop x is entered
// once, by a leg >= mi[x] (its cheapest incoming leg), and a closed tour
// still returns to the depot (>= the cheapest return leg); lb = that sum.
// int32: exact, prune iff key(prefix + lb) > bound. fp32: lb is summed and
// reduced with round-down, and a route continuing a prefix c with k more
// non-negative legs costs at least (c + sum)(1 - 2^-24)^k, so the test is
// RD(RD(c + lb) * (1 - 17 * 2^-24)) > bound (k <= 16) - still exact.
template <class C>
__device__ __forceinline__ uint32_t bb_sub(uint32_t lb, uint32_t m) {
    if constexpr (std::is_same<C, CostI32>::value) return lb - m;
    return __float_as_uint(__fsub_rd(__uint_as_float(lb), __uint_as_float(m)));
}
template <class C>
__device__ __forceinline__ bool bb_prune(uint32_t c, uint32_t lb, uint32_t bound_key) {
    if constexpr (std::is_same<C, CostI32>::value) return C::key(c + lb) > bound_key;
    const float low = __fmul_rd(__fadd_rd(__uint_as_float(c), __uint_as_float(lb)), 1.0f - 17.0f * 0x1p-24f);
    return low > __uint_as_float(bound_key);
}
template <class C, int L, bool CL, int SH, bool PR>
struct Dfs {
    __device__ __forceinline__ static void run(const uint32_t *Ds, int ns, uint32_t unused, int prev, uint32_t cost,
                                               Best &best, uint32_t &rank, uint32_t B, const uint32_t *mi = nullptr,
                                               uint32_t lb = 0) {
        uint32_t rem = unused;
        while (rem) {
            const int x = __ffs(rem) - 1;
            rem &= rem - 1;
            const uint32_t c2 = C::add(cost, DSL(prev * ns + x));
            uint32_t lb2 = 0;
            if constexpr (PR) lb2 = bb_sub<C>(lb, mi[x]);
            if (PR && bb_prune<C>(c2, lb2, min(B, best.key))) {
                rank += c_fact[L - 1];
                continue;
            }
            Dfs<C, L - 1, CL, SH, PR>::run(Ds, ns, unused & ~(1u << x), x, c2, best, rank, B, mi, lb2);
        }
    }
};
template <class C, bool CL, int SH, bool PR>
struct Dfs<C, 2, CL, SH, PR> {   // two stops left, a < b: leaves (a, b) then (b, a)
    __device__ __forceinline__ static void run(const uint32_t *Ds, int ns, uint32_t unused, int prev, uint32_t cost,
                                               Best &best, uint32_t &rank, uint32_t, const uint32_t * = nullptr,
                                               uint32_t = 0) {
        const int a = __ffs(unused) - 1;
        const int b = __ffs(unused & (unused - 1)) - 1;
        const uint32_t cab = C::add(C::add(cost, DSL(prev * ns + a)), DSL(a * ns + b));
        const uint32_t cba = C::add(C::add(cost, DSL(prev * ns + b)), DSL(b * ns + a));
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, b, cab), best, rank);
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, a, cba), best, rank);
    }
};
template <class C, bool CL, int SH, bool PR>
struct Dfs<C, 3, CL, SH, PR> {   // three stops left, a < b < c: the 6 leaves in lexicographic order, straight-line
    __device__ __forceinline__ static void run(const uint32_t *Ds, int ns, uint32_t unused, int prev, uint32_t cost,
                                               Best &best, uint32_t &rank, uint32_t, const uint32_t * = nullptr,
                                               uint32_t = 0) {
        const int a = __ffs(unused) - 1;
        const uint32_t u2 = unused & (unused - 1);
        const int b = __ffs(u2) - 1;
        const int c = __ffs(u2 & (u2 - 1)) - 1;
        const int p0 = prev * ns, a0 = a * ns, b0 = b * ns, c0 = c * ns;
        const uint32_t pa = C::add(cost, DSL(p0 + a)), pb = C::add(cost, DSL(p0 + b)), pc = C::add(cost, DSL(p0 + c));
        const uint32_t ab = C::add(pa, DSL(a0 + b)), ac = C::add(pa, DSL(a0 + c));
        const uint32_t ba = C::add(pb, DSL(b0 + a)), bc = C::add(pb, DSL(b0 + c));
        const uint32_t ca = C::add(pc, DSL(c0 + a)), cb = C::add(pc, DSL(c0 + b));
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, c, C::add(ab, DSL(b0 + c))), best, rank);   // a b c
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, b, C::add(ac, DSL(c0 + b))), best, rank);   // a c b
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, c, C::add(ba, DSL(a0 + c))), best, rank);   // b a c
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, a, C::add(bc, DSL(c0 + a))), best, rank);   // b c a
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, b, C::add(ca, DSL(a0 + b))), best, rank);   // c a b
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, a, C::add(cb, DSL(b0 + a))), best, rank);   // c b a
    }
};
template <class C, bool CL, int SH, bool PR>
struct Dfs<C, 1, CL, SH, PR> {
    __device__ __forceinline__ static void run(const uint32_t *Ds, int ns, uint32_t unused, int prev, uint32_t cost,
                                               Best &best, uint32_t &rank, uint32_t, const uint32_t * = nullptr,
                                               uint32_t = 0) {
        const int a = __ffs(unused) - 1;
        leaf<C>(ret_leg<C, CL, SH>(Ds, ns, a, C::add(cost, DSL(prev * ns + a))), best, rank);
    }
};

template <class C, bool CL, int SH, bool PR>
__device__ __forceinline__ void walk_subtree(int L, const uint32_t *Ds, int ns, uint32_t unused, int prev,
                                             uint32_t cost, Best &best, uint32_t &rank, uint32_t B,
                                             const uint32_t *mi = nullptr, uint32_t lb = 0) {
    switch (L) {
        case 1: Dfs<C, 1, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
        case 2: Dfs<C, 2, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
        case 3: Dfs<C, 3, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
        case 4: Dfs<C, 4, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
        case 5: Dfs<C, 5, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
        case 6: Dfs<C, 6, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
        default: Dfs<C, 7, CL, SH, PR>::run(Ds, ns, unused, prev, cost, best, rank, B, mi, lb); break;
    }
}

// One warp per work item (problem, prefix range). D submatrix staged in smem.
constexpr int ENUM_WARPS = 8;
// Branch and bound from this many stops (C4 exact, 11 stops: 81.5 -> 57 ms
// per step; 6-8-stop orders enumerate faster without the bound's divergence)
#ifndef ENUM_BB_MIN
#define ENUM_BB_MIN 9
#endif
// SH = 5: dynamic shared memory holds per warp ns_max^2 elements x 32 lane
// copies (large problems: 9-13 stops, where bank conflicts of a single copy
// dominate); SH = 0: one copy per warp (6-8 stops: occupancy matters more).
template <class C, int SH>
__global__ void __launch_bounds__(ENUM_WARPS * 32) route_enum_kernel(const RouteProblem *__restrict__ probs,
                                                                     const RouteWorkItem *__restrict__ items,
                                                                     int nitems, const uint32_t *__restrict__ Dall,
                                                                     uint64_t *item_best, int ns_max) {
    extern __shared__ uint32_t sDyn[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int it = blockIdx.x * ENUM_WARPS + warp;
    if (it >= nitems) return;
    const RouteWorkItem item = items[it];
    const RouteProblem pr = probs[item.problem];
    const int n = pr.n;
    const bool closed = pr.dep >= 0;
    const int ns = n + (closed ? 1 : 0);   // closed: local index n is the depot
    const uint32_t *D = Dall + (size_t)pr.order * DSTRIDE;
    uint32_t *Dw = sDyn + (size_t)warp * ns_max * ns_max * (SH ? 32 : 1);
    bool neg = false;   // int32: a negative or INF leg (prefix costs may then decrease or wrap)
    __shared__ uint32_t sMi[ENUM_WARPS][MS];
    uint32_t ret_min = 0;
    // stage: lane l loads element e = l, l + 32, ...; replicated: every
    // element is then broadcast to the 32 lane copies by a shuffle
    for (int e0 = 0; e0 < ns * ns; e0 += 32) {
        const int e = e0 + lane;
        uint32_t v = 0;
        if (e < ns * ns) {
            const int a = e / ns, b = e % ns;
            const int ia = a < n ? nib(pr.map, a) : pr.dep, ib = b < n ? nib(pr.map, b) : pr.dep;
            v = D[ia * MS + ib];
            neg |= std::is_same<C, CostI32>::value && ((int)v < 0 || v == CostI32::INF);
        }
        if constexpr (SH) {
            const int cnt = min(32, ns * ns - e0);
            for (int k = 0; k < cnt; ++k) Dw[(e0 + k) * 32 + lane] = __shfl_sync(0xffffffffu, v, k);
        } else if (e < ns * ns) {
            Dw[e] = v;
        }
    }
    __syncwarp();
    const uint32_t *Ds = Dw + (SH ? lane : 0);   // element e at Ds[e << SH]
    // branch and bound when every leg is >= 0: the bound B starts at the
    // best of 32 nearest-neighbour routes (lane l starts at stop l % n)
    const bool prune = n >= ENUM_BB_MIN && !__any_sync(0xffffffffu, neg);
    uint32_t B = 0xffffffffu;
    if (prune) {
        uint32_t unusedb = (1u << n) - 1u, cb = 0;
        int pv = closed ? n : -1;
        for (int a = 0; a < n; ++a) {
            int pick = -1;
            uint32_t pk = 0;
            if (a == 0) {
                pick = lane % n;
            } else {
                for (int x = 0; x < n; ++x) {   // nearest unvisited, ties -> smallest index
                    if (!((unusedb >> x) & 1u)) continue;
                    const uint32_t k = C::key(DSL(pv * ns + x));
                    if (pick < 0 || k < pk) { pick = x; pk = k; }
                }
            }
            if (pv >= 0) cb = C::add(cb, DSL(pv * ns + pick));
            unusedb &= ~(1u << pick);
            pv = pick;
        }
        if (closed) cb = C::add(cb, DSL(pv * ns + n));
        B = __reduce_min_sync(0xffffffffu, C::key(cb));
        {   // cheapest incoming leg per stop, cheapest return (int32 and fp32 >= 0: min of the bits)
            if (lane < n) {
                uint32_t m = 0xffffffffu;
                for (int y = 0; y < n; ++y)
                    if (y != lane) m = min(m, C::key(DSL(y * ns + lane)));
                sMi[warp][lane] = C::unkey(m);
            }
            uint32_t r = 0xffffffffu;
            if (closed && lane < n) r = C::key(DSL(lane * ns + n));
            ret_min = closed ? C::unkey(__reduce_min_sync(0xffffffffu, r)) : 0u;
            __syncwarp();
        }
    }
    const int p = prefix_depth(n);
    const int L = n - p;
    const uint32_t sub = c_fact[L];
    const uint32_t div0 = c_fact[n - 1] / sub;   // prefixes per first-element choice
    Best best{0xffffffffu, 0xffffffffu};
    for (int q0 = item.prefix_lo; q0 < item.prefix_hi; q0 += 32) {
        if (prune)   // share the lanes' best keys (all lanes reach this point together)
            B = min(B, __reduce_min_sync(0xffffffffu, best.key));
        const int q = q0 + lane;
        if (q >= item.prefix_hi) continue;
        // decode prefix q (mixed radix n, n-1, ..., n-p+1), lexicographic
        uint32_t unused = (1u << n) - 1u;
        uint32_t rem = (uint32_t)q, div = div0;
        int prev = closed ? n : -1;   // a closed tour leaves the depot first
        uint32_t cost = 0;
        for (int k = 0; k < p; ++k) {
            const uint32_t digit = rem / div;
            rem -= digit * div;
            if (k + 1 < p) div /= (uint32_t)(n - 1 - k);
            uint32_t m = unused;
            for (uint32_t t = 0; t < digit; ++t) m &= m - 1;
            const int x = __ffs(m) - 1;
            unused &= ~(1u << x);
            cost = prev >= 0 ? C::add(cost, DSL(prev * ns + x)) : cost;
            prev = x;
        }
        uint32_t rank = (uint32_t)q * sub;
        uint32_t lb = 0;
        if (prune) {
            lb = ret_min;
            for (uint32_t u2 = unused; u2; u2 &= u2 - 1) {
                const uint32_t m = sMi[warp][__ffs(u2) - 1];
                if constexpr (std::is_same<C, CostI32>::value) lb += m;
                else lb = __float_as_uint(__fadd_rd(__uint_as_float(lb), __uint_as_float(m)));
            }
        }
        if (prune && bb_prune<C>(cost, lb, min(B, best.key))) continue;   // the whole subtree
        if (prune) {
            if (closed) walk_subtree<C, true, SH, true>(L, Ds, ns, unused, prev, cost, best, rank, B, sMi[warp], lb);
            else walk_subtree<C, false, SH, true>(L, Ds, ns, unused, prev, cost, best, rank, B, sMi[warp], lb);
        } else {
            if (closed) walk_subtree<C, true, SH, false>(L, Ds, ns, unused, prev, cost, best, rank, B);
            else walk_subtree<C, false, SH, false>(L, Ds, ns, unused, prev, cost, best, rank, B);
        }
    }
    uint64_t packed = ((uint64_t)best.key << 32) | best.rank;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, packed, o);
        packed = y < packed ? y : packed;
    }
    if (lane == 0) item_best[it] = packed;
}

__global__ void problem_reduce_kernel(const RouteProblem *probs, int nprob, const uint64_t *item_best,
                                      uint64_t *prob_best) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nprob) return;
    uint64_t b = ~0ull;
    for (int k = probs[i].item0; k < probs[i].item0 + probs[i].nitems; ++k) b = item_best[k] < b ? item_best[k] : b;
    prob_best[i] = b;
}

// ------------------------------------------------- O8 segment plan (K-means) --
// Exact integer K-means with the tie rules of O8 (reading A12). With
// |coord| < 2^20 and n <= 16, (cnt*x - Sx)^2 * cnt'^2 < 2^63: int64 is exact.
__device__ inline int64_t sqd_scaled(int64_t x, int64_t y, int64_t sx, int64_t sy, int64_t cnt) {
    const int64_t dx = cnt * x - sx, dy = cnt * y - sy;
    return dx * dx + dy * dy;
}

__device__ void kmeans_dev(const int *xy, int n, int K, int *labels) {
    if (K > n) K = n;
    int centre[MS];
    centre[0] = 0;
    for (int k = 1; k < K; ++k) {
        int64_t best = -1;
        int arg = 0;
        for (int p = 0; p < n; ++p) {
            int64_t mind = -1;
            for (int q = 0; q < k; ++q) {
                const int64_t dx = (int64_t)xy[2 * p] - xy[2 * centre[q]];
                const int64_t dy = (int64_t)xy[2 * p + 1] - xy[2 * centre[q] + 1];
                const int64_t d = dx * dx + dy * dy;
                if (mind < 0 || d < mind) mind = d;
            }
            if (mind > best) {
                best = mind;
                arg = p;
            }
        }
        centre[k] = arg;
    }
    int64_t sx[MS], sy[MS], cnt[MS];
    for (int k = 0; k < K; ++k) {
        sx[k] = xy[2 * centre[k]];
        sy[k] = xy[2 * centre[k] + 1];
        cnt[k] = 1;
    }
    int prev[MS];
    bool have_prev = false;
    for (int it = 0; it < 100; ++it) {
        for (int p = 0; p < n; ++p) {
            int arg = 0;
            for (int k = 1; k < K; ++k) {
                const int64_t lhs = sqd_scaled(xy[2 * p], xy[2 * p + 1], sx[k], sy[k], cnt[k]) * (cnt[arg] * cnt[arg]);
                const int64_t rhs = sqd_scaled(xy[2 * p], xy[2 * p + 1], sx[arg], sy[arg], cnt[arg]) * (cnt[k] * cnt[k]);
                if (lhs < rhs) arg = k;
            }
            labels[p] = arg;
        }
        bool same = have_prev;
        for (int p = 0; p < n && same; ++p) same = prev[p] == labels[p];
        if (same) break;
        for (int p = 0; p < n; ++p) prev[p] = labels[p];
        have_prev = true;
        for (int k = 0; k < K; ++k) {
            int64_t nx = 0, ny = 0, c = 0;
            for (int p = 0; p < n; ++p)
                if (labels[p] == k) {
                    nx += xy[2 * p];
                    ny += xy[2 * p + 1];
                    ++c;
                }
            if (c > 0) {
                sx[k] = nx;
                sy[k] = ny;
                cnt[k] = c;
            }
        }
    }
}

__global__ void segment_plan_kernel(const int *xy, int n, int m, int *labels) {
    if (blockIdx.x == 0 && threadIdx.x == 0) kmeans_dev(xy, n, m, labels);
}

// --------------------------------------------------- a2 stop projection --
// Per order: distinct location nodes sorted ascending (P226-238 §2.4);
// status ETOOLARGE if more than 16 distinct stops. Marks source vertices.
// depot >= 0 (closed tours, NEXT-4): the depot joins every order's stop set
// (so it is a BF source and D holds its row and column); dep_info[o] = its
// index in the sorted stops | 256 if the order itself has a line there.
__global__ void order_stops_kernel(const int64_t *order_ptr, const int *nodes, int64_t B, int V, int *stops,
                                   int *n_out, int *status, int *is_src, int *bad, int depot, int *dep_info) {
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= B) return;
    int s[MS];
    int n = 0;
    int st = WR_OK;
    for (int64_t a = order_ptr[o]; a < order_ptr[o + 1]; ++a) {
        const int x = nodes[a];
        if (x < 0 || x >= V) {
            atomicOr(bad, 1);
            st = WR_EINVAL;
            break;
        }
        int pos = n;
        bool dup = false;
        for (int b = 0; b < n; ++b) {
            if (s[b] == x) { dup = true; break; }
        }
        if (dup) continue;
        if (n == MS) { st = WR_ETOOLARGE; break; }
        while (pos > 0 && s[pos - 1] > x) { s[pos] = s[pos - 1]; --pos; }
        s[pos] = x;
        ++n;
    }
    if (depot >= 0 && st == WR_OK) {
        int at = -1;
        for (int b = 0; b < n; ++b)
            if (s[b] == depot) at = b;
        const int genuine = at >= 0;
        if (!genuine) {
            if (n == MS) {
                st = WR_ETOOLARGE;
            } else {
                int pos = n;
                while (pos > 0 && s[pos - 1] > depot) { s[pos] = s[pos - 1]; --pos; }
                s[pos] = depot;
                at = pos;
                ++n;
            }
        }
        dep_info[o] = st == WR_OK ? (at | (genuine << 8)) : -1;
    } else if (dep_info) {
        dep_info[o] = -1;
    }
    for (int k = 0; k < MS; ++k) stops[o * MS + k] = k < n ? s[k] : -1;
    n_out[o] = n;
    status[o] = st;
    if (st == WR_OK)
        for (int k = 0; k < n; ++k) is_src[s[k]] = 1;
}

// Caller labels per order line -> per (order, stop) labels [B][16]: lines at
// the same node must agree (bad |= 2), labels must be >= 0 (bad |= 4).
__global__ void line_labels_kernel(const int64_t *order_ptr, const int *nodes, const int *line_labels, int64_t B,
                                   const int *stops, const int *n_arr, const int *status, int *lab, int *bad) {
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= B) return;
    int l[MS];
    for (int k = 0; k < MS; ++k) l[k] = -1;
    if (status[o] == WR_OK) {
        const int *s = stops + o * MS;
        const int n = n_arr[o];
        for (int64_t a = order_ptr[o]; a < order_ptr[o + 1]; ++a) {
            const int x = nodes[a], y = line_labels[a];
            if (y < 0) atomicOr(bad, 4);
            int i = 0;
            while (i < n && s[i] != x) ++i;
            if (i == n) continue;
            if (l[i] >= 0 && l[i] != y) atomicOr(bad, 2);
            l[i] = y;
        }
    }
    for (int k = 0; k < MS; ++k) lab[o * MS + k] = l[k] < 0 ? 0 : l[k];
}

__global__ void sources_scatter_kernel(const int *is_src, const int *src_row, int V, int *sources) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V && is_src[v]) sources[src_row[v]] = v;
}

__global__ void src_row_fix_kernel(const int *is_src, int *src_row, int V) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V && !is_src[v]) src_row[v] = -1;
}

// Ownership (a9): stops of order o owned by rank q form the contiguous index
// range [i_lo, i_hi) because stops are ascending and src_row is monotone.
__device__ inline void owned_range(const int *stops, int n, const int *src_row, int64_t lo, int64_t hi,
                                   int &i_lo, int &i_hi) {
    i_lo = 0;
    while (i_lo < n && src_row[stops[i_lo]] < lo) ++i_lo;
    i_hi = i_lo;
    while (i_hi < n && src_row[stops[i_hi]] < hi) ++i_hi;
}

__global__ void owned_count_kernel(const int *stops, const int *n_arr, const int *status, int64_t B,
                                   const int *src_row, const int64_t *blk, int world, int64_t *cnt) {
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= B) return;
    const int n = status[o] == WR_OK ? n_arr[o] : 0;
    for (int q = 0; q < world; ++q) {
        int a, b;
        owned_range(stops + o * MS, n, src_row, blk[q], blk[q + 1], a, b);
        cnt[(int64_t)q * (B + 1) + o] = (int64_t)(b - a) * n;
    }
}

// a5 D gather: send[off[o] + (i - i_lo) * n + j] = dist(stop_i -> stop_j) for
// the stops i whose source row lies in this BF segment [seg_lo, seg_hi).
__global__ void gather_send_kernel(const int *stops, const int *n_arr, const int *status, int64_t B,
                                   const int *src_row, int64_t own_lo, int64_t own_hi, int64_t seg_lo,
                                   int64_t seg_hi, const int64_t *off, const uint32_t *rows, int V, int tsw,
                                   int pack, const int *pos_of, uint32_t *send) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= B * MS) return;
    const int64_t o = t / MS;
    const int i = (int)(t % MS);
    if (status[o] != WR_OK) return;
    const int n = n_arr[o];
    if (i >= n) return;
    const int *s = stops + o * MS;
    const int64_t r = src_row[s[i]];
    if (r < seg_lo || r >= seg_hi) return;
    int i_lo, i_hi;
    owned_range(s, n, src_row, own_lo, own_hi, i_lo, i_hi);
    const int64_t rr = pos_of[r - seg_lo];   // slot position of the source in the segment's tiles
    uint32_t *dst = send + off[o] + (int64_t)(i - i_lo) * n;
    if (pack >= 2) {   // packed u16 rows: widen, INF 0x7fff -> INT32_MAX; keyed rows (3): d = key >> 4
        const uint16_t *R = reinterpret_cast<const uint16_t *>(rows) + (size_t)(rr / tsw) * V * tsw + (rr % tsw);
        const int sh = pack == 3 ? 4 : 0;
        for (int j = 0; j < n; ++j) {
            const uint32_t x = R[(size_t)s[j] * tsw];
            dst[j] = x == 0x7fffu ? 0x7fffffffu : x >> sh;
        }
        return;
    }
    const uint32_t *R = rows + (size_t)(rr / tsw) * V * tsw + (rr % tsw);
    for (int j = 0; j < n; ++j) dst[j] = R[(size_t)s[j] * tsw];
}

// Reassemble D[o][i][j] (16 x 16 stride) for orders [o_lo, o_hi) from the
// all-gathered send buffers (rank-major, max_send elements each).
__global__ void assemble_kernel(const int *stops, const int *n_arr, const int *status, int64_t B, int64_t o_lo,
                                int64_t o_hi, const int *src_row, const int64_t *blk, int world,
                                const int64_t *off_all, const uint32_t *gathered, int64_t max_send,
                                uint32_t *Dall) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (o_hi - o_lo) * MS) return;
    const int64_t o = o_lo + t / MS;
    const int i = (int)(t % MS);
    uint32_t *D = Dall + (size_t)(o - o_lo) * DSTRIDE + i * MS;
    if (status[o] != WR_OK) return;
    const int n = n_arr[o];
    if (i >= n) return;
    const int *s = stops + o * MS;
    const int64_t r = src_row[s[i]];
    int q = 0;
    while (q + 1 < world && r >= blk[q + 1]) ++q;
    int i_lo, i_hi;
    owned_range(s, n, src_row, blk[q], blk[q + 1], i_lo, i_hi);
    const uint32_t *src = gathered + (int64_t)q * max_send + off_all[(int64_t)q * (B + 1) + o] + (int64_t)(i - i_lo) * n;
    for (int j = 0; j < n; ++j) D[j] = src[j];
}

// ------------------------------------------------ route preparation --
constexpr int PAIRS_MAX_SEG = 9;                  // stops per segment, boundary-pair mode
constexpr int64_t PAIRS_MAX_CAND = 1ll << 26;      // stitch candidates per order

struct OrderRoute {        // per-order routing state (device)
    int n;
    int status;
    int mseg;              // segments m' (1 = exact)
    int prob0;             // first problem index
    int nprob;
    uint64_t segmap[WR_MAX_SEGMENTS];  // nibble map of each segment's stops
    int seglen[WR_MAX_SEGMENTS];
    int hk;                // exact route of 13-16 stops by route_hk_kernel (NEXT-2)
    int noenum;            // no enumeration problems (Held-Karp or boundary-pair stitch)
    int dep;               // closed tour (NEXT-4): order-stop index of the depot; -1 open
    int ng;                // stops routed (the order's own: n, or n - 1 without a line at the depot)
    uint64_t gmap;         // nibble list of those ng order-stop indices (ascending)
};

template <class C>
__device__ inline bool is_inf(uint32_t x) { return x == C::INF; }

// Pass 1: status, segments, problem/item counts.
template <class C>
__global__ void route_prepare_kernel(const int *n_arr, const int *status_in, const int *stops, int64_t o_lo,
                                     int64_t nord, const uint32_t *Dall, int m, const int *xy,
                                     const int *labels_in, int64_t chunk, OrderRoute *ordr, int *prob_cnt,
                                     int *item_cnt, int pairs, int *hk_count, int *hk_list, const int *dep_info,
                                     int *shk_list) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nord) return;
    const int64_t o = o_lo + t;
    OrderRoute R;
    R.n = n_arr[o];
    R.status = status_in[o];
    R.mseg = 1;
    R.prob0 = 0;
    R.nprob = 0;
    R.hk = 0;
    R.noenum = 0;
    int nitems = 0;
    const int n = R.n;
    // closed tours (NEXT-4): the depot sits among the n stops of D; the
    // routed stops are the order's own (the depot only if it has a line there)
    const int di = dep_info ? dep_info[o] : -1;
    R.dep = di >= 0 ? (di & 0xff) : -1;
    const bool dep_routed = di >= 0 && (di >> 8);
    int gs[MS], ng = 0;
    for (int i = 0; i < n; ++i)
        if (R.dep < 0 || i != R.dep || dep_routed) gs[ng++] = i;
    R.ng = ng;
    R.gmap = 0;
    for (int a = 0; a < ng; ++a) R.gmap |= (uint64_t)gs[a] << (4 * a);
    if (R.status == WR_OK) {
        const uint32_t *D = Dall + (size_t)t * DSTRIDE;
        for (int i = 0; i < n && R.status == WR_OK; ++i)
            for (int j = 0; j < n; ++j)
                if (i != j && is_inf<C>(D[i * MS + j])) { R.status = WR_EUNREACHABLE; break; }
    }
    if (R.status == WR_OK) {
        int lab[MS];   // per routed stop (a = 0..ng-1 <-> order stop gs[a])
        if (m <= 1 || ng <= 1) {
            for (int a = 0; a < ng; ++a) lab[a] = 0;
        } else if (labels_in) {
            for (int a = 0; a < ng; ++a) lab[a] = labels_in[t * MS + gs[a]];
        } else {
            int pxy[2 * MS];
            const int *s = stops + o * MS;
            for (int a = 0; a < ng; ++a) {
                pxy[2 * a] = xy[2 * s[gs[a]]];
                pxy[2 * a + 1] = xy[2 * s[gs[a]] + 1];
            }
            kmeans_dev(pxy, ng, m, lab);
        }
        // relabel by first appearance (O7 step 1)
        int map_lab[MS], nseg = 0, seg_of[MS];
        for (int a = 0; a < ng; ++a) {
            int id = -1;
            for (int k = 0; k < nseg; ++k)
                if (map_lab[k] == lab[a]) id = k;
            if (id < 0) {
                if (nseg == WR_MAX_SEGMENTS) { R.status = WR_ETOOLARGE; break; }
                map_lab[nseg] = lab[a];
                id = nseg++;
            }
            seg_of[a] = id;
        }
        if (R.status == WR_OK) {
            R.mseg = nseg > 0 ? nseg : 1;
            for (int k = 0; k < WR_MAX_SEGMENTS; ++k) { R.seglen[k] = 0; R.segmap[k] = 0; }
            for (int a = 0; a < ng; ++a) {
                const int k = seg_of[a];
                R.segmap[k] |= (uint64_t)gs[a] << (4 * R.seglen[k]);
                R.seglen[k]++;
            }
            if (nseg == 1 && ng >= SHK_MIN && ng <= SHK_MAX && shk_list) {
                // exact route of an 8-stop order: warp Held-Karp (route_hk_small_kernel)
                R.hk = 2;
                R.noenum = 1;
                nseg = 0;
                shk_list[atomicAdd(hk_count + 4, 1)] = (int)t;
            }
            if (nseg == 1 && ng > WR_MAX_EXACT) {
                // exact route of 13-16 stops: Held-Karp subset DP (NEXT-2)
                R.hk = 1;
                R.noenum = 1;
                nseg = 0;
                hk_list[atomicAdd(hk_count, 1)] = (int)t;   // [0] count, [2] max routed stops
                atomicMax(hk_count + 2, ng);
            }
            if (pairs && nseg >= 2) {
                // boundary-pair stitch (NEXT-1): per-segment orders and the
                // stitch run in the finalize warp; limits as the oracle's
                int64_t ncand = fact(nseg);
                for (int k = 0; k < nseg; ++k) {
                    const int nj = R.seglen[k];
                    if (nj > PAIRS_MAX_SEG) R.status = WR_ETOOLARGE;
                    ncand *= nj >= 2 ? (int64_t)nj * (nj - 1) : 1;
                }
                if (ncand > PAIRS_MAX_CAND) R.status = WR_ETOOLARGE;
                R.noenum = 1;
                nseg = 0;   // no enumeration problems
            }
            for (int k = 0; k < nseg; ++k) {
                if (R.seglen[k] > WR_MAX_EXACT) { R.status = WR_ETOOLARGE; break; }
                if (R.seglen[k] >= 2) {
                    const int nj = R.seglen[k];
                    atomicMax(hk_count + 3, nj + (nseg == 1 && R.dep >= 0 ? 1 : 0));   // enum staging size
                    const int p = prefix_depth(nj);
                    const int64_t npre = fact(nj) / fact(nj - p);
                    const int64_t per = chunk / fact(nj - p) > 0 ? chunk / fact(nj - p) : 1;
                    R.nprob++;
                    nitems += (int)((npre + per - 1) / per);
                }
            }
        }
    }
    if (R.status != WR_OK) { R.nprob = 0; nitems = 0; }
    ordr[t] = R;
    prob_cnt[t] = R.nprob;
    item_cnt[t] = nitems;
}

// Pass 2: emit problems and work items at the scanned offsets.
__global__ void route_emit_kernel(int64_t nord, OrderRoute *ordr, const int *prob_off, const int *item_off,
                                  int64_t chunk, RouteProblem *probs, RouteWorkItem *items) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nord) return;
    OrderRoute &R = ordr[t];
    R.prob0 = prob_off[t];
    if (R.status != WR_OK || R.noenum) return;   // counted no problems (prepare)
    int pi = prob_off[t], ii = item_off[t];
    for (int k = 0; k < R.mseg; ++k) {
        const int nj = R.seglen[k];
        if (nj < 2) continue;
        const int p = prefix_depth(nj);
        const int npre = (int)(fact(nj) / fact(nj - p));
        const int64_t per64 = chunk / fact(nj - p) > 0 ? chunk / fact(nj - p) : 1;
        const int per = (int)(per64 < npre ? per64 : npre);
        RouteProblem P;
        P.order = (int)t;
        P.n = nj;
        P.dep = R.mseg == 1 ? R.dep : -1;   // segments of a stitched tour stay open (reading R4)
        P.map = R.segmap[k];
        P.item0 = ii;
        P.nitems = (npre + per - 1) / per;
        for (int q = 0; q < npre; q += per) {
            RouteWorkItem W;
            W.problem = pi;
            W.prefix_lo = q;
            W.prefix_hi = q + per < npre ? q + per : npre;
            items[ii++] = W;
        }
        probs[pi++] = P;
    }
}

// Finalise: warp per order. Exact: unrank the best; segmented: stitch the
// m'! 2^m' oriented concatenations (O7 step 3-4) with a full left-to-right
// recompute, ties -> lexicographically smallest sequence.
template <class C>
__global__ void route_finalize_kernel(int64_t nord, const OrderRoute *ordr, const uint64_t *prob_best,
                                      const RouteProblem *probs, const uint32_t *Dall, const int *stops,
                                      int64_t o_lo, wr_route_result *out, unsigned long long *counters, int pairs) {
    __shared__ uint32_t sD[4][DSTRIDE];
    __shared__ unsigned long long s_perms;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t = (int64_t)blockIdx.x * 4 + warp;
    if (threadIdx.x == 0) s_perms = 0;
    __syncthreads();
    do {   // one exit: the block adds its routes-covered count with one atomic
    if (t >= nord) break;
    const OrderRoute R = ordr[t];
    const int n = R.ng;   // stops routed (closed tours: without a depot that has no line)
    const int *s = stops + (o_lo + t) * MS;
    wr_route_result res;
    res.n = n;
    res.status = R.status;
    res.m_used = R.mseg;
    res.rank = 0;
    res.cost_bits = C::INF;
    for (int k = 0; k < MS; ++k) res.seq[k] = -1;
    if (R.status != WR_OK) {
        if (lane == 0) out[t] = res;
        break;
    }
    if (pairs && R.mseg >= 2) break;   // route_pairs_kernel writes these orders
    if (R.hk) break;                   // route_hk_kernel / route_hk_small_kernel write these orders
    const int dep = R.dep;              // closed tour (NEXT-4): the depot's stop index, else -1
    const uint32_t *D = Dall + (size_t)t * DSTRIDE;
    uint32_t *Ds = sD[warp];
    if (R.mseg >= 2 || (n < 2 && dep >= 0)) {   // only the stitch and an out-and-back read D here
        for (int e = lane; e < DSTRIDE; e += 32) Ds[e] = D[e];
        __syncwarp();
    }
    uint64_t final_seq = 0;
    uint32_t final_cost = 0;
    unsigned long long perms = 0;
    // each segment's best route as a nibble sequence of order-stop indices
    uint64_t segseq[WR_MAX_SEGMENTS];
    int pi = R.prob0;
    for (int k = 0; k < R.mseg; ++k) {
        const int nj = R.seglen[k];
        if (nj >= 2) {
            const uint64_t b = prob_best[pi];
            const uint64_t loc = unrank_nib((int64_t)(uint32_t)b, nj);
            uint64_t g = 0;
            for (int a = 0; a < nj; ++a) g |= (uint64_t)nib(R.segmap[k], nib(loc, a)) << (4 * a);
            segseq[k] = g;
            perms += (unsigned long long)fact(nj);
            ++pi;
        } else {
            segseq[k] = R.segmap[k];   // 0 or 1 stop
        }
    }
    if (R.mseg == 1) {
        final_seq = segseq[0];
        if (n >= 2) {
            final_cost = C::unkey((uint32_t)(prob_best[R.prob0] >> 32));   // the closed cost for closed problems
        } else if (dep >= 0) {   // one stop: out and back
            final_cost = C::add(Ds[dep * MS + nib(final_seq, 0)], Ds[nib(final_seq, 0) * MS + dep]);
        } else {
            final_cost = 0u;
        }
    } else {
        const int m = R.mseg;
        const int64_t ncand = fact(m) << m;
        uint32_t best_key = 0xffffffffu;
        uint64_t best_seq = ~0ull;
        for (int64_t c = lane; c < ncand; c += 32) {
            const uint64_t tau = unrank_nib(c >> m, m);
            const int bits = (int)(c & ((1 << m) - 1));
            uint64_t seq = 0;
            int pos = 0;
            for (int k = 0; k < m; ++k) {
                const int j = nib(tau, k);
                const int nj = R.seglen[j];
                const bool rev = (bits >> k) & 1;
                for (int a = 0; a < nj; ++a) {
                    const int x = nib(segseq[j], rev ? nj - 1 - a : a);
                    seq |= (uint64_t)x << (4 * pos);
                    ++pos;
                }
            }
            // full left-to-right recompute; a closed tour starts with the
            // depot leg and ends with the return leg (reading R4)
            uint32_t cost = dep >= 0 ? C::add(Ds[dep * MS + nib(seq, 0)], Ds[nib(seq, 0) * MS + nib(seq, 1)])
                                     : Ds[nib(seq, 0) * MS + nib(seq, 1)];
            for (int a = 2; a < n; ++a) cost = C::add(cost, Ds[nib(seq, a - 1) * MS + nib(seq, a)]);
            if (dep >= 0) cost = C::add(cost, Ds[nib(seq, n - 1) * MS + dep]);
            const uint32_t key = C::key(cost);
            // lexicographic key: first stop in the most significant nibble
            uint64_t lex = 0;
            for (int a = 0; a < n; ++a) lex |= (uint64_t)nib(seq, a) << (4 * (15 - a));
            if (key < best_key || (key == best_key && lex < best_seq)) {
                best_key = key;
                best_seq = lex;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint32_t k2 = __shfl_xor_sync(0xffffffffu, best_key, o);
            const uint64_t s2 = __shfl_xor_sync(0xffffffffu, best_seq, o);
            if (k2 < best_key || (k2 == best_key && s2 < best_seq)) {
                best_key = k2;
                best_seq = s2;
            }
        }
        final_cost = C::unkey(best_key);
        final_seq = 0;
        for (int a = 0; a < n; ++a) final_seq |= (uint64_t)((best_seq >> (4 * (15 - a))) & 0xf) << (4 * a);
        if (lane == 0) atomicAdd(&counters[1], (unsigned long long)ncand);
    }
    if (lane == 0) {
        // Lehmer rank of the final sequence among the n! orders
        int64_t rank = 0;
        for (int a = 0; a < n; ++a) {
            int smaller = 0;
            for (int b = a + 1; b < n; ++b) smaller += nib(final_seq, b) < nib(final_seq, a);
            rank += smaller * fact(n - 1 - a);
        }
        res.rank = rank;
        res.cost_bits = (n >= 2 || dep >= 0) ? final_cost : 0u;
        for (int a = 0; a < n; ++a) res.seq[a] = s[nib(final_seq, a)];
        out[t] = res;
        atomicAdd(&s_perms, perms);
    }
    } while (false);
    __syncthreads();
    if (threadIdx.x == 0 && s_perms) atomicAdd(&counters[0], s_perms);
}

// NEXT-1 boundary-pair stitch (WR_ROUTE_PAIRS; oracle:
// orc_segmented_pairs_route): one block per order, so a segment of up to 9
// stops (9! local orders) is enumerated by PAIRS_THREADS threads.
constexpr int PAIRS_THREADS = 256;
template <class C>
__global__ void __launch_bounds__(PAIRS_THREADS) route_pairs_kernel(int64_t nord, const OrderRoute *ordr,
                                                                    const uint32_t *Dall, const int *stops,
                                                                    int64_t o_lo, wr_route_result *out,
                                                                    unsigned long long *counters) {
    __shared__ uint32_t Ds[DSTRIDE];
    // best (cost key << 32 | local lexicographic rank) per (segment, first,
    // last), then the kept path as a nibble sequence of order stops
    __shared__ unsigned long long sPair[WR_MAX_SEGMENTS][PAIRS_MAX_SEG][PAIRS_MAX_SEG];
    __shared__ uint32_t sBestKey[PAIRS_THREADS / 32];
    __shared__ uint64_t sBestSeq[PAIRS_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t = blockIdx.x;
    if (t >= nord) return;
    const OrderRoute R = ordr[t];
    if (R.status != WR_OK || R.mseg < 2) return;   // route_finalize_kernel writes these
    const int n = R.ng;     // stops routed
    const int dep = R.dep;  // closed tour (NEXT-4): the depot's stop index, else -1
    const int *s = stops + (o_lo + t) * MS;
    const uint32_t *D = Dall + (size_t)t * DSTRIDE;
    for (int e = tid; e < DSTRIDE; e += PAIRS_THREADS) Ds[e] = D[e];
    unsigned long long perms = 0;
    {
        // NEXT-1 boundary-pair stitch (oracle: orc_segmented_pairs_route).
        // 1. per segment, every local order (lexicographic rank r) is costed
        //    left to right; its (first, last) bin keeps the smallest
        //    (cost key, r) - ties -> the lexicographically smallest order
        const int m = R.mseg;
        unsigned long long(*tab)[PAIRS_MAX_SEG][PAIRS_MAX_SEG] = sPair;
        for (int k = 0; k < m; ++k)
            for (int e = tid; e < PAIRS_MAX_SEG * PAIRS_MAX_SEG; e += PAIRS_THREADS)
                tab[k][e / PAIRS_MAX_SEG][e % PAIRS_MAX_SEG] = ~0ull;
        __syncthreads();
        for (int k = 0; k < m; ++k) {
            const int nj = R.seglen[k];
            if (nj < 2) continue;
            const int64_t nf = fact(nj);
            perms += (unsigned long long)nf;
            // each thread walks a contiguous rank range: one unrank, then
            // lexicographic successors (next permutation) - no per-order
            // 64-bit divisions
            const int64_t per = (nf + PAIRS_THREADS - 1) / PAIRS_THREADS;
            const int64_t r0 = (int64_t)tid * per, r1 = r0 + per < nf ? r0 + per : nf;
            if (r0 < r1) {
                int loc[PAIRS_MAX_SEG], stp[PAIRS_MAX_SEG];
                const uint64_t l0 = unrank_nib(r0, nj);
                for (int a = 0; a < nj; ++a) loc[a] = nib(l0, a);
                for (int a = 0; a < nj; ++a) stp[a] = nib(R.segmap[k], a);
                for (int64_t r = r0;;) {
                    int prev = stp[loc[0]];
                    int x = stp[loc[1]];
                    uint32_t cost = Ds[prev * MS + x];
                    prev = x;
                    for (int a = 2; a < nj; ++a) {
                        x = stp[loc[a]];
                        cost = C::add(cost, Ds[prev * MS + x]);
                        prev = x;
                    }
                    const unsigned long long key = ((unsigned long long)C::key(cost) << 32) | (unsigned long long)r;
                    atomicMin(&tab[k][loc[0]][loc[nj - 1]], key);
                    if (++r >= r1) break;
                    int i = nj - 2;   // next permutation of loc (lexicographic)
                    while (loc[i] > loc[i + 1]) --i;
                    int j = nj - 1;
                    while (loc[j] < loc[i]) --j;
                    const int tmp = loc[i];
                    loc[i] = loc[j];
                    loc[j] = tmp;
                    for (int a = i + 1, b = nj - 1; a < b; ++a, --b) {
                        const int t2 = loc[a];
                        loc[a] = loc[b];
                        loc[b] = t2;
                    }
                }
            }
        }
        __syncthreads();
        // 2. the kept path of every pair as a nibble sequence of order stops
        for (int k = 0; k < m; ++k) {
            const int nj = R.seglen[k];
            for (int e = tid; e < nj * nj; e += PAIRS_THREADS) {
                const int a = e / nj, b = e % nj;
                uint64_t g = 0;
                if (nj == 1) {
                    g = R.segmap[k];
                } else if (a != b) {
                    const uint64_t loc = unrank_nib((int64_t)(uint32_t)tab[k][a][b], nj);
                    for (int t2 = 0; t2 < nj; ++t2) g |= (uint64_t)nib(R.segmap[k], nib(loc, t2)) << (4 * t2);
                }
                tab[k][a][b] = g;
            }
        }
        __syncthreads();
        // 3. stitch: segment order x one endpoint pair per segment, full
        //    left-to-right recompute, ties -> lexicographically smallest
        int np[WR_MAX_SEGMENTS];
        uint32_t P = 1;   // <= PAIRS_MAX_CAND: 32-bit index arithmetic
        for (int k = 0; k < m; ++k) {
            const int nj = R.seglen[k];
            np[k] = nj >= 2 ? nj * (nj - 1) : 1;
            P *= (uint32_t)np[k];
        }
        const uint32_t ncand = (uint32_t)fact(m) * P;
        uint32_t best_key = 0xffffffffu;
        uint64_t best_seq = ~0ull;
        for (uint32_t c = tid; c < ncand; c += PAIRS_THREADS) {
            const uint64_t tau = unrank_nib((int64_t)(c / P), m);
            uint32_t rest = c % P;
            uint64_t seq = 0;
            int pos = 0;
            for (int k = m - 1; k >= 0; --k) {   // mixed radix, last segment fastest
                const int j = nib(tau, k);
                const int nj = R.seglen[j];
                const int p = (int)(rest % (uint32_t)np[j]);
                rest /= (uint32_t)np[j];
                int a = 0, b = 0;
                if (nj >= 2) {
                    a = p / (nj - 1);
                    b = p % (nj - 1);
                    b += b >= a;
                }
                // place segment k's path at its position: positions are
                // filled right to left (segments k+1.. already placed)
                pos += nj;
                seq |= tab[j][a][b] << (4 * (n - pos));
            }
            // full left-to-right recompute; a closed tour starts with the
            // depot leg and ends with the return leg (reading R4)
            uint32_t cost = dep >= 0 ? C::add(Ds[dep * MS + nib(seq, 0)], Ds[nib(seq, 0) * MS + nib(seq, 1)])
                                     : Ds[nib(seq, 0) * MS + nib(seq, 1)];
            for (int a = 2; a < n; ++a) cost = C::add(cost, Ds[nib(seq, a - 1) * MS + nib(seq, a)]);
            if (dep >= 0) cost = C::add(cost, Ds[nib(seq, n - 1) * MS + dep]);
            const uint32_t key = C::key(cost);
            uint64_t lex = 0;
            for (int a = 0; a < n; ++a) lex |= (uint64_t)nib(seq, a) << (4 * (15 - a));
            if (key < best_key || (key == best_key && lex < best_seq)) {
                best_key = key;
                best_seq = lex;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint32_t k2 = __shfl_xor_sync(0xffffffffu, best_key, o);
            const uint64_t s2 = __shfl_xor_sync(0xffffffffu, best_seq, o);
            if (k2 < best_key || (k2 == best_key && s2 < best_seq)) {
                best_key = k2;
                best_seq = s2;
            }
        }
        if (lane == 0) {
            sBestKey[warp] = best_key;
            sBestSeq[warp] = best_seq;
        }
        __syncthreads();
        if (tid != 0) return;
        for (int w2 = 1; w2 < PAIRS_THREADS / 32; ++w2)
            if (sBestKey[w2] < best_key || (sBestKey[w2] == best_key && sBestSeq[w2] < best_seq)) {
                best_key = sBestKey[w2];
                best_seq = sBestSeq[w2];
            }
        const uint32_t final_cost = C::unkey(best_key);
        uint64_t final_seq = 0;
        for (int a = 0; a < n; ++a) final_seq |= (uint64_t)((best_seq >> (4 * (15 - a))) & 0xf) << (4 * a);
        atomicAdd(&counters[1], (unsigned long long)ncand);
        int64_t rank = 0;   // Lehmer rank of the final sequence among the n! orders
        for (int a = 0; a < n; ++a) {
            int smaller = 0;
            for (int b2 = a + 1; b2 < n; ++b2) smaller += nib(final_seq, b2) < nib(final_seq, a);
            rank += smaller * fact(n - 1 - a);
        }
        wr_route_result res;
        res.n = n;
        res.status = WR_OK;
        res.m_used = m;
        res.rank = rank;
        res.cost_bits = final_cost;
        for (int a = 0; a < MS; ++a) res.seq[a] = a < n ? s[nib(final_seq, a)] : -1;
        out[t] = res;
        atomicAdd(&counters[0], perms);

    }
}

// NEXT-2 exact route for 13-16 stops (oracle: orc_held_karp_route, reading
// R2): O5's result - the minimum left-to-right cost, ties -> the
// lexicographically smallest order - in three passes over cost-only state
// tables W[S][j] (S = stop set, j = last stop, row stride 16):
//  1. forward subset DP F(S, j) = min_i fl(F(S-j, i) + D[i][j]) -> C*;
//  2. backward bound M(S, j) = the largest prefix cost with which some
//     completion still ends <= C*: M(all, j) = C*, M(S, j) = max over
//     unvisited k of inv(D[j][k], M(S+k, k)), inv(d, m) = max{c : fl(c + d)
//     <= m} (written over F, layer by layer);
//  3. lexicographic greedy: next stop = the smallest k with fl(c + D[j][k])
//     <= M(S+k, k).
// One order per 8-CTA cluster: a layer's states are split over the cluster's
// 4,096 threads and layers are separated by cluster barriers; the subsets of
// each popcount come from a precomputed list. At most HK_CLUSTERS tables of
// 2^n x 16 x 4 B (4 MB at n = 16) are live, so they stay in L2; workspace
// loads/stores bypass L1 (ld/st .cg).
constexpr int HK_THREADS = 512;
constexpr int HK_CL = 8;            // CTAs per cluster (one order each)
constexpr int HK_CLUSTERS = 18;     // clusters in flight: 144 SMs, 72 MB of tables
constexpr int HK_MAX = WR_MAX_STOPS;
constexpr int LIST_MIN = 7;          // popcount-sorted subset lists are kept for n = 7..16
constexpr int HK_RS = 16;           // workspace row stride (states of one S)

// fp32: max{c >= 0 : fl(c + d) <= m} exactly (RN-even), -1 if none. fl(x) <=
// m iff x < T or (x == T and m's significand is even), T = m + ulp(m)/2 (the
// midpoint to the next float; exact in double); c is the largest float below
// T - d (or equal to it when the tie goes to m): directed double subtraction,
// then directed conversion.
__device__ inline float f32_inv(float d, float m) {
    if (!(d <= m)) return -1.0f;                       // even c = 0 gives fl(d) > m
    if (isinf(m)) return __int_as_float(0x7f800000);
    const uint32_t mb = __float_as_uint(m);
    const int e = (int)(mb >> 23);
    // half an ulp of m: 2^(e - 151) for normal m, 2^-150 for subnormal (built directly)
    const double half = __longlong_as_double((long long)((e > 0 ? e : 1) - 151 + 1023) << 52);
    const double T = (double)m + half;
    const double lo = __dsub_rd(T, (double)d), hi = __dsub_ru(T, (double)d);
    float c = __double2float_rd(lo);
    if ((mb & 1u) && lo == hi && (double)c == lo) c = __uint_as_float(__float_as_uint(c) - 1u);   // strict
    return c;
}

template <class C>
struct HkOps;
template <>
struct HkOps<CostI32> {    // int32 (sums exact within the route bound, A7)
    static constexpr uint32_t NONE = 0x80000000u;
    __device__ static uint32_t fwd(uint32_t pre, uint32_t leg) {
        return (pre == CostI32::INF || leg == CostI32::INF) ? CostI32::INF : (uint32_t)((int)pre + (int)leg);
    }
    // max c with c + leg <= m, saturated to int32 (prefix sums stay strictly
    // inside (INT32_MIN, INT32_MAX), so saturation never changes a test)
    __device__ static uint32_t inv(uint32_t leg, uint32_t m) {
        if (leg == CostI32::INF || m == NONE) return NONE;
        int64_t c = (int64_t)(int)m - (int)leg;
        if (c >= (int64_t)INT32_MAX) c = INT32_MAX - 1;
        if (c <= (int64_t)INT32_MIN) return NONE;
        return (uint32_t)(int)c;
    }
    __device__ static bool gt(uint32_t a, uint32_t b) { return (int)a > (int)b; }   // NONE is the least
    __device__ static bool step(uint32_t c, uint32_t leg, uint32_t m, uint32_t &out) {
        if (m == NONE || leg == CostI32::INF) return false;
        const int64_t x = (int64_t)(int)c + (int)leg;
        out = (uint32_t)(int)x;
        return x <= (int64_t)(int)m;
    }
};
template <>
struct HkOps<CostF32> {    // fp32 >= 0; NONE = -1.0f
    static constexpr uint32_t NONE = 0xbf800000u;
    __device__ static uint32_t fwd(uint32_t pre, uint32_t leg) { return CostF32::add(pre, leg); }
    __device__ static uint32_t inv(uint32_t leg, uint32_t m) {
        if (m == NONE) return NONE;
        return __float_as_uint(f32_inv(__uint_as_float(leg), __uint_as_float(m)));
    }
    __device__ static bool gt(uint32_t a, uint32_t b) { return __uint_as_float(a) > __uint_as_float(b); }
    __device__ static bool step(uint32_t c, uint32_t leg, uint32_t m, uint32_t &out) {
        if (m == NONE) return false;
        out = CostF32::add(c, leg);
        return __uint_as_float(out) <= __uint_as_float(m);
    }
};

struct HkLists {           // subsets of [0, n) sorted by popcount, n = LIST_MIN..16
    const uint16_t *sets;  // concatenated lists
    int off[HK_MAX - LIST_MIN + 1][HK_MAX + 2];   // [n - LIST_MIN][k] start of popcount k
};

template <class C>
__global__ void __cluster_dims__(HK_CL, 1, 1) __launch_bounds__(HK_THREADS)
    route_hk_kernel(const int *__restrict__ hk_list, int nhk, const OrderRoute *ordr, const uint32_t *Dall,
                    const int *stops, int64_t o_lo, wr_route_result *out, unsigned long long *counters,
                    int *next, uint32_t *ws, size_t ws_stride, HkLists L) {
    namespace cg = cooperative_groups;
    using H = HkOps<C>;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned crank = cl.block_rank();
    const int tid = threadIdx.x;
    const int gtid = (int)crank * HK_THREADS + tid, gstride = HK_CL * HK_THREADS;
    __shared__ uint32_t Ds[DSTRIDE];
    __shared__ uint32_t DsT[MS * (MS + 1)];   // DsT[j * 17 + i] = D[i][j] (conflict-free column reads)
    __shared__ uint32_t Din[MS], Dout[MS];   // closed tour (NEXT-4): the depot legs
    __shared__ int s_i, s_slow;
    uint32_t *W = ws + (size_t)(blockIdx.x / HK_CL) * ws_stride;
    for (;;) {
        if (crank == 0 && tid == 0) s_i = atomicAdd(next, 1);
        cl.sync();
        const int i = *cl.map_shared_rank(&s_i, 0);
        cl.sync();   // every CTA has read rank 0's claim
        if (i >= nhk) break;
        const int t = hk_list[i];
        const OrderRoute R = ordr[t];
        const int n = R.ng;   // stops routed; local stop a is order stop nib(R.gmap, a)
        const bool closed = R.dep >= 0;
        const uint32_t *D = Dall + (size_t)t * DSTRIDE;
        if (tid == 0) s_slow = 0;
        __syncthreads();
        // int32 fast path: every leg finite and |leg| < 2^23, so prefix sums
        // and bounds stay within +-2^29 and absent terms can be padded with
        // +-2^30 instead of tested (results identical to the general path)
        const auto leg_slow = [&](uint32_t v) {
            if (!std::is_same<C, CostI32>::value) return false;
            return v == C::INF || (int)v >= (1 << 23) || (int)v <= -(1 << 23);
        };
        for (int e = tid; e < DSTRIDE; e += HK_THREADS) {
            const int a = e / MS, b = e % MS;
            const uint32_t v = (a < n && b < n) ? D[nib(R.gmap, a) * MS + nib(R.gmap, b)] : 0u;
            Ds[e] = v;
            DsT[b * (MS + 1) + a] = v;
            if (leg_slow(v)) s_slow = 1;
        }
        if (closed && tid < n) {
            Din[tid] = D[R.dep * MS + nib(R.gmap, tid)];
            Dout[tid] = D[nib(R.gmap, tid) * MS + R.dep];
            if (leg_slow(Din[tid]) || leg_slow(Dout[tid])) s_slow = 1;
        }
        const uint16_t *sets = L.sets;
        const int *off = L.off[n - LIST_MIN];
        __syncthreads();
        const bool fast = std::is_same<C, CostI32>::value && !s_slow;   // same in every CTA of the cluster
        // F({j}, j) = 0, or the depot leg of a closed tour
        if (gtid < n) __stcg(W + (size_t)(1u << gtid) * HK_RS + gtid, closed ? Din[gtid] : 0u);
        __syncthreads();
        cl.sync();
        // 1. forward layers |S| = 2..n, one item per (P, j): P of layer
        //    |S| - 1, j not in P, S = P + j. Consecutive items share P (one
        //    row fetch per warp), the column D[.][j] comes from DsT, and the
        //    row's absent entries are masked (never read by the oracle's
        //    min, reading R2): INF for fp32 (fl(INF + d) = INF is the
        //    largest key; D is never -0), +2^30 on the int fast path
        const uint32_t full = (1u << n) - 1u;
        for (int k = 2; k <= n; ++k) {
            const int pb = off[k - 1], fan = n - k + 1, items = (off[k] - pb) * fan;
            for (int x = gtid; x < items; x += gstride) {
                const int pidx = x / fan, b = x - pidx * fan;
                const uint32_t P = sets[pb + pidx];
                const int j = __fns(~P & full, 0, b + 1);
                const uint32_t *dcol = DsT + j * (MS + 1);
                const uint4 *row = reinterpret_cast<const uint4 *>(W + (size_t)P * HK_RS);
                uint32_t r[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 v = __ldcg(row + q);
                    r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
                }
                uint32_t outv;
                if (fast) {
                    int bi = 0x7fffffff;
#pragma unroll
                    for (int a2 = 0; a2 < 16; ++a2) {
                        const int ra = ((P >> a2) & 1u) ? (int)r[a2] : (1 << 30);
                        bi = min(bi, ra + (int)dcol[a2]);
                    }
                    outv = (uint32_t)bi;
                } else if (std::is_same<C, CostF32>::value) {
                    uint32_t best = 0xffffffffu;
#pragma unroll
                    for (int a2 = 0; a2 < 16; ++a2) {
                        const uint32_t ra = ((P >> a2) & 1u) ? r[a2] : CostF32::INF;
                        best = min(best, C::key(H::fwd(ra, dcol[a2])));
                    }
                    outv = C::unkey(best);
                } else {
                    uint32_t best = 0xffffffffu;
#pragma unroll
                    for (int a2 = 0; a2 < 16; ++a2)
                        if ((P >> a2) & 1u) best = min(best, C::key(H::fwd(r[a2], dcol[a2])));
                    outv = C::unkey(best);
                }
                __stcg(W + (size_t)(P | (1u << j)) * HK_RS + j, outv);
            }
            cl.sync();
        }
        // C* = min over the last stop of F(all, j) (+ the return leg)
        const uint32_t F = (1u << n) - 1u;
        uint32_t ck = 0xffffffffu;
        for (int j = 0; j < n; ++j) {
            const uint32_t f = __ldcg(W + (size_t)F * HK_RS + j);
            ck = min(ck, C::key(closed ? H::fwd(f, Dout[j]) : f));
        }
        const uint32_t cstar = C::unkey(ck);
        cl.sync();   // every CTA has C* before M(all, .) overwrites F(all, .)
        wr_route_result res;
        if (cstar == C::INF) {   // every order costs INF: O5 keeps the identity (rank 0)
            if (crank == 0 && tid == 0) {
                const int *s = stops + (o_lo + t) * MS;
                res.n = n;
                res.status = WR_OK;
                res.m_used = 1;
                res.cost_bits = C::INF;
                res.rank = 0;
                for (int a = 0; a < MS; ++a) res.seq[a] = a < n ? s[nib(R.gmap, a)] : -1;
                out[t] = res;
            }
            cl.sync();
            continue;
        }
        // 2. backward bound, layers |S| = n .. 1 (closed: the largest prefix
        //    whose return leg still ends <= C*)
        if (gtid < n) __stcg(W + (size_t)F * HK_RS + gtid, closed ? H::inv(Dout[gtid], cstar) : cstar);
        cl.sync();
        for (int k = n - 1; k >= 1; --k) {
            const int base = off[k], items = (off[k + 1] - base) * k;
            for (int x = gtid; x < items; x += gstride) {
                const int sidx = x / k, b = x - sidx * k;
                const uint32_t S = sets[base + sidx];
                const int j = __fns(S, 0, b + 1);
                const uint32_t rest = F & ~S;
                // every successor bound loaded before any is used (independent
                // loads instead of a chain of L2 round trips); one thread per
                // set instead (loads shared by the set's k states) was slower:
                // 26.0 vs 30.4 k orders/s at 16 stops, too little parallelism
                uint32_t mv[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    mv[q] = ((rest >> q) & 1u) ? __ldcg(W + (size_t)(S | (1u << q)) * HK_RS + q) : H::NONE;
                uint32_t best = H::NONE;
                if (fast) {   // NONE -> -2^30: its c stays below -2^29, every real c above
                    int bi = -(1 << 30) - (1 << 24);
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int m = mv[q] == H::NONE ? -(1 << 30) : (int)mv[q];
                        bi = max(bi, m - (int)Ds[j * MS + q]);
                    }
                    best = bi < -(1 << 29) ? H::NONE : (uint32_t)bi;
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        if (!((rest >> q) & 1u)) continue;
                        const uint32_t c = H::inv(Ds[j * MS + q], mv[q]);
                        if (H::gt(c, best)) best = c;
                    }
                }
                __stcg(W + (size_t)S * HK_RS + j, best);
            }
            cl.sync();
        }
        // 3. lexicographic greedy (one warp: lane q tests stop q, the
        //    smallest passing lane is the pick - one L2 round trip per step)
        if (crank == 0 && tid < 32) {
            const int lane = tid;
            uint32_t S = 0, c = 0;
            int j = -1, seq[MS];
            bool ok = true;
            for (int a = 0; a < n && ok; ++a) {
                bool pass = false;
                uint32_t nx = 0;
                if (lane < n && !((S >> lane) & 1u)) {
                    const uint32_t m = __ldcg(W + (size_t)(S | (1u << lane)) * HK_RS + lane);
                    if (a == 0) {   // the first stop's prefix: 0, or the depot leg
                        nx = closed ? Din[lane] : 0u;
                        pass = m != H::NONE && !H::gt(nx, m);
                    } else {
                        pass = H::step(c, Ds[j * MS + lane], m, nx);
                    }
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, pass);
                ok = bal != 0u;
                if (!ok) break;
                const int pick = __ffs(bal) - 1;
                c = __shfl_sync(0xffffffffu, nx, pick);
                seq[a] = pick;
                S |= 1u << pick;
                j = pick;
            }
            if (lane == 0) {
                if (ok && closed) c = H::fwd(c, Dout[j]);   // the return leg
                const int *s = stops + (o_lo + t) * MS;
                res.n = n;
                res.status = ok ? WR_OK : WR_EINTERNAL;
                res.m_used = 1;
                res.cost_bits = c;
                int64_t rank = 0;   // Lehmer rank among the n! orders
                for (int a = 0; a < n && ok; ++a) {
                    int smaller = 0;
                    for (int b = a + 1; b < n; ++b) smaller += seq[b] < seq[a];
                    rank += smaller * fact(n - 1 - a);
                }
                res.rank = rank;
                for (int a = 0; a < MS; ++a) res.seq[a] = (ok && a < n) ? s[nib(R.gmap, seq[a])] : -1;
                out[t] = res;
                // work: forward transitions n (n-1) 2^(n-2), as many in the bound pass
                atomicAdd(&counters[0], 2ull * (unsigned long long)n * (n - 1) * (1ull << (n - 2)));
            }
        }
        cl.sync();   // the table is reused by the cluster's next order
    }
}

// Exact routes of SHK_MIN..SHK_MAX stops (default 8) by the same three
// passes as route_hk_kernel (forward DP, backward bound, lexicographic
// greedy: O5's answer, reading R2), one warp per order with its table in
// shared memory (2^n x 8 words). An 8-stop order costs n 2^(n-1) = 1,024
// states per pass here against 8! = 40,320 enumerated leaves; at 7 stops and
// below enumeration is as cheap, so those stay with route_enum_kernel.
static_assert(SHK_MIN >= LIST_MIN && SHK_MAX <= 8, "warp Held-Karp: 7 <= n <= 8");
constexpr int SHK_WARPS = 8;
constexpr int SHK_RS = 8;   // table row stride (n <= 8)
constexpr size_t SHK_SMEM = (size_t)SHK_WARPS * ((1u << SHK_MAX) * SHK_RS + 64 + 16) * sizeof(uint32_t);

template <class C>
__global__ void __launch_bounds__(SHK_WARPS * 32)
    route_hk_small_kernel(const int *__restrict__ list, int nlist, const OrderRoute *ordr, const uint32_t *Dall,
                          const int *stops, int64_t o_lo, wr_route_result *out, unsigned long long *counters,
                          HkLists L) {
    using H = HkOps<C>;
    extern __shared__ uint32_t shk[];
    __shared__ unsigned long long s_routes;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * SHK_WARPS + warp;
    if (threadIdx.x == 0) s_routes = 0;
    __syncthreads();
    do {   // one exit: the block adds its routes-covered count with one atomic
    if (i >= nlist) break;
    uint32_t *W = shk + (size_t)warp * ((1u << SHK_MAX) * SHK_RS + 64 + 16);
    uint32_t *Ds = W + (1u << SHK_MAX) * SHK_RS;   // [a * 8 + b]
    uint32_t *Din = Ds + 64, *Dout = Din + 8;
    const int t = list[i];
    const OrderRoute R = ordr[t];
    const int n = R.ng;
    const bool closed = R.dep >= 0;
    const uint32_t *D = Dall + (size_t)t * DSTRIDE;
    for (int e = lane; e < 64; e += 32) {
        const int a = e >> 3, b = e & 7;
        Ds[e] = (a < n && b < n) ? D[nib(R.gmap, a) * MS + nib(R.gmap, b)] : 0u;
    }
    if (closed && lane < n) {
        Din[lane] = D[R.dep * MS + nib(R.gmap, lane)];
        Dout[lane] = D[nib(R.gmap, lane) * MS + R.dep];
    }
    __syncwarp();
    // int32 fast path (as route_hk_kernel): every leg finite and |leg| < 2^23,
    // so F and M stay within +-2^29 and the INF / NONE tests can go
    bool slow = false;
    if (std::is_same<C, CostI32>::value) {
        const auto bad = [](uint32_t v) { return v == C::INF || (int)v >= (1 << 23) || (int)v <= -(1 << 23); };
        for (int e = lane; e < 64; e += 32) slow |= ((e >> 3) < n && (e & 7) < n) && bad(Ds[e]);
        if (closed && lane < n) slow |= bad(Din[lane]) || bad(Dout[lane]);
    }
    const bool fast = std::is_same<C, CostI32>::value && !__any_sync(0xffffffffu, slow);
    const uint16_t *sets = L.sets;
    const int *off = L.off[n - LIST_MIN];
    if (lane < n) W[(1u << lane) * SHK_RS + lane] = closed ? Din[lane] : 0u;
    __syncwarp();
    // 1. forward: F(S, j) = min over i in S - j of fl(F(S - j, i) + D[i][j])
    for (int k = 2; k <= n; ++k) {
        const int base = off[k], items = (off[k + 1] - base) * k;
        const float rk = 1.0f / (float)k;
        for (int x = lane; x < items; x += 32) {
            const int sidx = (int)(((float)x + 0.5f) * rk), b = x - sidx * k;   // x < 2^10: exact
            const uint32_t S = sets[base + sidx];
            const int j = __fns(S, 0, b + 1);
            const uint32_t P = S & ~(1u << j);
            if (fast) {
                int bi = 0x7fffffff;
                for (uint32_t q = P; q; q &= q - 1) {
                    const int a = __ffs(q) - 1;
                    bi = min(bi, (int)W[P * SHK_RS + a] + (int)Ds[a * 8 + j]);
                }
                W[S * SHK_RS + j] = (uint32_t)bi;
                continue;
            }
            uint32_t best = 0xffffffffu;
            for (uint32_t q = P; q; q &= q - 1) {
                const int a = __ffs(q) - 1;
                best = min(best, C::key(H::fwd(W[P * SHK_RS + a], Ds[a * 8 + j])));
            }
            W[S * SHK_RS + j] = C::unkey(best);
        }
        __syncwarp();
    }
    const uint32_t F = (1u << n) - 1u;
    uint32_t ck = 0xffffffffu;
    if (lane < n) {
        const uint32_t f = W[F * SHK_RS + lane];
        ck = C::key(closed ? H::fwd(f, Dout[lane]) : f);
    }
    const uint32_t cstar = C::unkey(__reduce_min_sync(0xffffffffu, ck));
    const int *s = stops + (o_lo + t) * MS;
    wr_route_result res;
    if (cstar == C::INF) {   // every order costs INF: O5 keeps the identity (rank 0)
        if (lane == 0) {
            res.n = n;
            res.status = WR_OK;
            res.m_used = 1;
            res.cost_bits = C::INF;
            res.rank = 0;
            for (int a = 0; a < MS; ++a) res.seq[a] = a < n ? s[nib(R.gmap, a)] : -1;
            out[t] = res;
        }
        break;
    }
    // 2. backward bound M(S, j), written over F layer by layer
    __syncwarp();
    if (lane < n) W[F * SHK_RS + lane] = closed ? H::inv(Dout[lane], cstar) : cstar;
    __syncwarp();
    for (int k = n - 1; k >= 1; --k) {
        const int base = off[k], items = (off[k + 1] - base) * k;
        const float rk = 1.0f / (float)k;
        for (int x = lane; x < items; x += 32) {
            const int sidx = (int)(((float)x + 0.5f) * rk), b = x - sidx * k;   // x < 2^10: exact
            const uint32_t S = sets[base + sidx];
            const int j = __fns(S, 0, b + 1);
            if (fast) {   // NONE -> -2^30: its c stays below -2^29, every real c above
                int bi = -(1 << 30) - (1 << 24);
                for (uint32_t q = F & ~S; q; q &= q - 1) {
                    const int a = __ffs(q) - 1;
                    const uint32_t mv = W[(S | (1u << a)) * SHK_RS + a];
                    bi = max(bi, (mv == H::NONE ? -(1 << 30) : (int)mv) - (int)Ds[j * 8 + a]);
                }
                W[S * SHK_RS + j] = bi < -(1 << 29) ? H::NONE : (uint32_t)bi;
                continue;
            }
            uint32_t best = H::NONE;
            for (uint32_t q = F & ~S; q; q &= q - 1) {
                const int a = __ffs(q) - 1;
                const uint32_t c = H::inv(Ds[j * 8 + a], W[(S | (1u << a)) * SHK_RS + a]);
                if (H::gt(c, best)) best = c;
            }
            W[S * SHK_RS + j] = best;
        }
        __syncwarp();
    }
    // 3. lexicographic greedy: lane q tests stop q, the smallest passing lane wins
    uint32_t Sv = 0, c = 0;
    int j = -1, seq[MS];
    bool ok = true;
    for (int a = 0; a < n && ok; ++a) {
        bool pass = false;
        uint32_t nx = 0;
        if (lane < n && !((Sv >> lane) & 1u)) {
            const uint32_t m = W[(Sv | (1u << lane)) * SHK_RS + lane];
            if (a == 0) {
                nx = closed ? Din[lane] : 0u;
                pass = m != H::NONE && !H::gt(nx, m);
            } else {
                pass = H::step(c, Ds[j * 8 + lane], m, nx);
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, pass);
        ok = bal != 0u;
        if (!ok) break;
        const int pick = __ffs(bal) - 1;
        c = __shfl_sync(0xffffffffu, nx, pick);
        seq[a] = pick;
        Sv |= 1u << pick;
        j = pick;
    }
    if (lane == 0) {
        if (ok && closed) c = H::fwd(c, Dout[j]);   // the return leg
        res.n = n;
        res.status = ok ? WR_OK : WR_EINTERNAL;
        res.m_used = 1;
        res.cost_bits = c;
        int64_t rank = 0;   // Lehmer rank among the n! orders
        for (int a = 0; a < n && ok; ++a) {
            int smaller = 0;
            for (int b = a + 1; b < n; ++b) smaller += seq[b] < seq[a];
            rank += smaller * fact(n - 1 - a);
        }
        res.rank = rank;
        for (int a = 0; a < MS; ++a) res.seq[a] = (ok && a < n) ? s[nib(R.gmap, seq[a])] : -1;
        out[t] = res;
        atomicAdd(&s_routes, (unsigned long long)fact(n));   // routes covered, as enumeration counts them
    }
    } while (false);
    __syncthreads();
    if (threadIdx.x == 0 && s_routes) atomicAdd(&counters[0], s_routes);
}

// The popcount-sorted subset lists for n = 7..16 (host-built once per
// device; 256 KB).
static HkLists hk_lists(int device) {
    static std::vector<std::pair<int, HkLists>> cache;
    static std::vector<DBuf<uint16_t>> keep;
    for (auto &e : cache)
        if (e.first == device) return e.second;
    HkLists L{};
    std::vector<uint16_t> all;
    for (int n = LIST_MIN; n <= HK_MAX; ++n) {
        int *off = L.off[n - LIST_MIN];
        for (int k = 0; k <= n; ++k) {
            off[k] = (int)all.size();
            for (uint32_t S = 0; S < (1u << n); ++S)
                if (__builtin_popcount(S) == k) all.push_back((uint16_t)S);
        }
        off[n + 1] = (int)all.size();
    }
    DBuf<uint16_t> d;
    {
        StreamScope s0(0);   // process-lifetime buffer on the legacy stream
        d = to_device<uint16_t>(all.data(), all.size(), 0);
        WR_CUDA(cudaStreamSynchronize(0));
    }
    L.sets = d.p;
    keep.push_back(std::move(d));
    cache.push_back({device, L});
    return L;
}

// ------------------------------------------------------ route_cost (O4) --
template <class C>
__global__ void route_cost_kernel(const uint32_t *D, int n, const int *seqs, int len, int64_t count,
                                  uint32_t *costs, int *bad) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const int *s = seqs + t * len;
    for (int a = 0; a < len; ++a)
        if (s[a] < 0 || s[a] >= n) { atomicOr(bad, 1); return; }
    if (len < 2) { costs[t] = 0u; return; }
    bool inf = false;
    uint32_t c = D[s[0] * n + s[1]];
    int64_t ci = (int)c;
    inf = c == C::INF;
    for (int a = 2; a < len; ++a) {
        const uint32_t leg = D[s[a - 1] * n + s[a]];
        inf |= leg == C::INF;
        c = C::add(c, leg);
        ci += (int)leg;
    }
    if (C::INF == 0x7fffffffu) {     // int32: exact sum, INF legs -> INF
        if (inf) c = C::INF;
        else if (ci >= (int64_t)INT32_MAX || ci < (int64_t)INT32_MIN) { atomicOr(bad, 2); return; }
        else c = (uint32_t)(int)ci;
    }
    costs[t] = c;
}

// =========================================================== host side ==
struct Plan {               // wr_plan
    int device = 0;
    const wr_graph *g = nullptr;
    int64_t B = 0, S = 0;
    int rank = 0, world = 1;
    int64_t src_lo = 0, src_hi = 0, order_lo = 0, order_hi = 0;
    int64_t send_count = 0, max_send = 0;
    int m = 1;
    int pairs = 0;          // WR_ROUTE_PAIRS: boundary-pair stitch (NEXT-1)
    int64_t chunk = WR_DEFAULT_CHUNK;
    DBuf<int> stops, n_arr, status, is_src, src_row, sources;
    DBuf<int64_t> blk;      // world+1 source block boundaries
    DBuf<int64_t> off_all;  // world x (B+1)
    DBuf<int> labels;       // optional [B][16] labels override
    DBuf<int> dep_info;     // closed tours: [B] depot stop index | 256 if a genuine stop; -1 open
    int closed = 0;
    std::vector<int64_t> h_blk;
    int64_t launches = 0;
};

}  // namespace wr

struct wr_plan : wr::Plan {};

namespace wr {

static unsigned gridn(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static wr_status plan_impl(const wr_graph *g, const int64_t *order_ptr, const int32_t *order_nodes, int64_t B,
                           int32_t rank, int32_t world, const wr_route_opts *opts, const int32_t *labels16,
                           const int32_t *line_labels,
                           wr_plan **out) {
    if (!g || !out || B < 0 || (B > 0 && (!order_ptr || !order_nodes)))
        return fail(WR_EINVAL, "wr_orders_plan: bad arguments");
    if (world < 1 || rank < 0 || rank >= world) return fail(WR_EINVAL, "wr_orders_plan: rank/world");
    WR_CUDA(cudaSetDevice(g->device));
    const int64_t l0 = g_launches;
    wr_route_opts o{};
    if (opts) o = *opts;
    cudaStream_t st = (cudaStream_t)o.stream;
    StreamScope stream_scope(st);
    auto P = std::make_unique<wr_plan>();
    P->device = g->device;
    P->g = g;
    P->B = B;
    P->rank = rank;
    P->world = world;
    P->m = (line_labels && o.m < 2) ? 2 : o.m;   // caller labels always go through the stitch
    P->pairs = (o.flags & WR_ROUTE_PAIRS) ? 1 : 0;
    P->chunk = o.chunk > 0 ? o.chunk : WR_DEFAULT_CHUNK;
    P->closed = (o.flags & WR_ROUTE_CLOSED) ? 1 : 0;
    if (P->closed && (o.depot < 0 || o.depot >= g->V)) return fail(WR_EINVAL, "wr_orders_plan: depot outside [0, V)");
    if (P->m >= 2 && !labels16 && !g->xy.p)
        return fail(WR_EINVAL, "wr_orders_plan: segmented routing without labels needs graph xy (O8)");
    const int V = g->V;
    int64_t L = 0;
    if (B > 0) {
        WR_CUDA(cudaMemcpy(&L, order_ptr + B, 8, cudaMemcpyDefault));
        int64_t first = 0;
        WR_CUDA(cudaMemcpy(&first, order_ptr, 8, cudaMemcpyDefault));
        if (first != 0 || L < 0) return fail(WR_EINVAL, "wr_orders_plan: order_ptr must start at 0");
    }
    DBuf<int64_t> d_ptr = to_device<int64_t>(order_ptr, B + 1, st);
    DBuf<int> d_nodes = to_device<int>(order_nodes, L, st);
    P->stops.alloc(std::max<int64_t>(B, 1) * WR_MAX_STOPS);
    P->n_arr.alloc(std::max<int64_t>(B, 1));
    P->status.alloc(std::max<int64_t>(B, 1));
    P->is_src.alloc(V);
    P->src_row.alloc(V);
    DBuf<int> bad(1);
    WR_CUDA(cudaMemsetAsync(P->is_src.p, 0, 4LL * V, st));
    WR_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
    if (P->closed) P->dep_info.alloc(std::max<int64_t>(B, 1));
    if (B > 0) {
        order_stops_kernel<<<gridn(B, 256), 256, 0, st>>>(d_ptr.p, d_nodes.p, B, V, P->stops.p, P->n_arr.p,
                                                         P->status.p, P->is_src.p, bad.p,
                                                         P->closed ? o.depot : -1, P->dep_info.p);
        count_launch();
        WR_LAUNCH_CHECK();
    }
    if (line_labels && B > 0) {
        DBuf<int> d_ll = to_device<int>(line_labels, L, st);
        P->labels.alloc((size_t)B * WR_MAX_STOPS);
        line_labels_kernel<<<gridn(B, 256), 256, 0, st>>>(d_ptr.p, d_nodes.p, d_ll.p, B, P->stops.p, P->n_arr.p,
                                                         P->status.p, P->labels.p, bad.p);
        count_launch();
        WR_LAUNCH_CHECK();
    }
    int hbad = 0;
    WR_CUDA(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    if (hbad & 1) return fail(WR_EINVAL, "wr_orders_plan: order node outside [0, V)");
    if (hbad & 2) return fail(WR_EINVAL, "wr_orders_plan: lines at the same node carry different labels");
    if (hbad & 4) return fail(WR_EINVAL, "wr_orders_plan: negative label");
    scan_exclusive_i32(P->is_src.p, P->src_row.p, V, st);
    int last_row = 0, last_flag = 0;
    WR_CUDA(cudaMemcpyAsync(&last_row, P->src_row.p + V - 1, 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaMemcpyAsync(&last_flag, P->is_src.p + V - 1, 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    P->S = (int64_t)last_row + last_flag;
    P->sources.alloc(std::max<int64_t>(P->S, 1));
    sources_scatter_kernel<<<gridn(V, 256), 256, 0, st>>>(P->is_src.p, P->src_row.p, V, P->sources.p);
    src_row_fix_kernel<<<gridn(V, 256), 256, 0, st>>>(P->is_src.p, P->src_row.p, V);
    count_launch();
    count_launch();
    WR_LAUNCH_CHECK();
    // source blocks and order blocks
    P->h_blk.resize(world + 1);
    for (int q = 0; q < world; ++q) {
        int64_t lo, hi;
        wr_shard_range(P->S, q, world, &lo, &hi);
        P->h_blk[q] = lo;
        P->h_blk[q + 1] = hi;
    }
    P->src_lo = P->h_blk[rank];
    P->src_hi = P->h_blk[rank + 1];
    wr_shard_range(B, rank, world, &P->order_lo, &P->order_hi);
    P->blk = to_device<int64_t>(P->h_blk.data(), world + 1, st);
    // per-rank owned-entry offsets: exclusive scans of counts over orders
    P->off_all.alloc((size_t)world * (B + 1));
    WR_CUDA(cudaMemsetAsync(P->off_all.p, 0, sizeof(int64_t) * world * (B + 1), st));
    if (B > 0) {
        owned_count_kernel<<<gridn(B, 256), 256, 0, st>>>(P->stops.p, P->n_arr.p, P->status.p, B, P->src_row.p,
                                                         P->blk.p, world, P->off_all.p);
        count_launch();
        WR_LAUNCH_CHECK();
    }
    std::vector<int64_t> totals(world);
    for (int q = 0; q < world; ++q) {
        int64_t *row = P->off_all.p + (int64_t)q * (B + 1);
        scan_exclusive_i64(row, row, B + 1, st);
        WR_CUDA(cudaMemcpyAsync(&totals[q], row + B, 8, cudaMemcpyDeviceToHost, st));
    }
    WR_CUDA(cudaStreamSynchronize(st));
    P->send_count = totals[rank];
    P->max_send = std::max<int64_t>(1, *std::max_element(totals.begin(), totals.end()));
    if (labels16) P->labels = to_device<int>(labels16, (size_t)std::max<int64_t>(B, 1) * WR_MAX_STOPS, st);
    WR_CUDA(cudaStreamSynchronize(st));
    P->launches = g_launches - l0;
    *out = P.release();
    return WR_OK;
}

// A second, libwr-owned stream per (host thread, device) for the sweep's
// concurrent tail part (event-ordered against the caller's stream).
static cudaStream_t side_stream(int device) {
    thread_local std::vector<std::pair<int, cudaStream_t>> cache;
    for (auto &e : cache)
        if (e.first == device) return e.second;
    cudaStream_t s = nullptr;
    WR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cache.push_back({device, s});
    return s;
}

static wr_status local_impl(wr_plan *P, void *send, const wr_route_opts *opts, wr_route_stats *stats) {
    if (!P || (!send && P->send_count > 0)) return fail(WR_EINVAL, "wr_orders_local: bad arguments");
    if (!is_device_ptr(send) && P->send_count > 0) return fail(WR_EINVAL, "wr_orders_local: send must be device memory");
    const wr_graph *g = P->g;
    WR_CUDA(cudaSetDevice(P->device));
    const int64_t l0 = g_launches;
    wr_route_opts o{};
    if (opts) o = *opts;
    cudaStream_t st = (cudaStream_t)o.stream;
    StreamScope stream_scope(st);
    const int V = g->V;
    const int64_t nsrc = P->src_hi - P->src_lo;
    const auto hstart = std::chrono::steady_clock::now();
    auto hms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hstart).count(); };
    cudaEvent_t e0, e1;
    WR_CUDA(cudaEventCreate(&e0));
    WR_CUDA(cudaEventCreate(&e1));
    WR_CUDA(cudaEventRecord(e0, st));
    BfTileStats h0{0ull, 0, -1, 0ull};
    DBuf<BfTileStats> d_stats(1);
    WR_CUDA(cudaMemcpyAsync(d_stats.p, &h0, sizeof(h0), cudaMemcpyHostToDevice, st));
    int segments = 0;
    float bf_ms = 0.f, pred_ms = 0.f;
    if (o.pred_out && (!is_device_ptr(o.pred_out) || o.pred_rows < P->src_hi - P->src_lo))
        return fail(WR_EINVAL, "wr_orders_local: pred_out must be device memory with >= src_hi-src_lo rows");
    // Packed u16 rows (OpU16) when every distance provably fits: int32
    // weights in [1, 0x3fff] (w > 0 also rules out flat vertices). A tile
    // whose distances approach 0x7fff raises the overflow flag and the whole
    // phase is redone with 32-bit rows.
    static const bool no_pack = getenv("WR_NO_PACK") != nullptr;
    int pack = (g->wtype == WR_I32 && !g->has_negative && !g->has_zero && g->max_abs_w <= 0x3fff && !no_pack &&
                !(o.flags & WR_ROUTE_ROWS32))
                   ? 2
                   : 1;
    // Keyed packed rows (OpK16) when the fused pred is requested: the pred
    // rides in the row keys (in-degree <= 15, w <= 0x7ff; d < 0x7ff, else
    // the overflow flag redoes the phase with plain packed rows).
    static const bool no_key = getenv("WR_NO_KEYED") != nullptr;
    const bool fused_req = o.pred_out && !g->has_negative && getenv("WR_NO_FUSED_PRED") == nullptr;
    bool keyed = pack == 2 && fused_req && !no_key && g->max_abs_w <= 0x7ff && g->max_in_deg <= 15;
    BfTileStats hs{};
    int64_t tiles_swept = 0;
    int tile_width = 0;
    auto run_phase = [&](int pk) {
        if (nsrc <= 0) return;
        wr_graph_info_t gi;
        wr_graph_info(g, &gi);
        const int64_t fixed = gi.device_bytes + (128 << 20);
        int nsm = 0;
        WR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
        const int spl = choose_spl(nsrc, nsm, pk);
        const int tsw = 32 * spl * pk;            // sources per tile
        const int64_t src_bytes = 4LL * V / pk;   // row bytes per source
        const double h_pre = hms();
        const int64_t budget = budget_bytes(o.hbm_budget, fixed, (nsrc + tsw - 1) / tsw * tsw * src_bytes);
        const double h_budget = hms();
        const int64_t sb = sources_per_segment(budget, fixed, src_bytes, nsrc, tsw);
        const int64_t tile_bytes = 4LL * V * 32 * spl;
        const int64_t max_tiles = tiles_to_allocate(sb, tsw, budget - fixed - sb * src_bytes, tile_bytes);
        static const bool trace = getenv("WR_TRACE") != nullptr;
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        if (trace) {
            WR_CUDA(cudaEventCreate(&t0));
            WR_CUDA(cudaEventCreate(&t1));
            WR_CUDA(cudaEventRecord(t0, st));
        }
        const auto hclock0 = std::chrono::steady_clock::now();
        // a4 fused into the sweep (non-negative weights): done list + counters
        static const bool no_fuse = getenv("WR_NO_FUSED_PRED") != nullptr;
        const bool fused = o.pred_out && !g->has_negative && !no_fuse;
        const int max_rounds = std::max(1, V - 1);   // + the kernel's check round (ENEGCYCLE if it changes)
        const int64_t *off_r = P->off_all.p + (int64_t)P->rank * (P->B + 1);
        cudaEvent_t b0, b1, b2;
        WR_CUDA(cudaEventCreate(&b0));
        WR_CUDA(cudaEventCreate(&b1));
        WR_CUDA(cudaEventCreate(&b2));
        // The sweep's makespan is ~ waves x tile time (one tile per SM at a
        // time): 331 tiles of 256 on 148 SMs leave 113 SMs to the fused
        // pred jobs through a third wave (C5 trace: 57 ms, 41 ms of sweep
        // work per SM). WR_TAIL_SPLIT=1: with packed rows and a single budget
        // segment, the sources beyond the last full wave of wide tiles go to
        // narrow tiles (64-wide: ~half the tile time) swept concurrently on
        // a second stream, launched first.
        // Measured on C5 (profiles/r02_tail_split.txt): the split ends the
        // last wide tile at 54 ms instead of 57, but the fused pred jobs,
        // which ran on the SMs the third wave left idle, then run after it:
        // the step got slower (76 vs 70 ms). Kept as an opt-in experiment.
        static const bool no_tail = getenv("WR_TAIL_SPLIT") == nullptr;
        struct Part {
            int64_t lo, hi;
            int spl;
        };
        std::vector<Part> parts;
        const bool single = sb >= nsrc;
        {
            const int64_t full_waves = (nsrc / tsw) / nsm;
            const int64_t main_n = full_waves * nsm * tsw;
            const int64_t rem = nsrc - main_n;
            if (single && pk == 2 && !no_tail && full_waves >= 1 && rem > 0) {
                int tspl = 1;   // the narrowest tile width whose tiles fit one wave
                while (tspl < spl && (rem + 32LL * tspl * pk - 1) / (32LL * tspl * pk) > nsm) tspl *= 2;
                parts.push_back({P->src_lo + main_n, P->src_hi, tspl});   // tail first: its CTAs start first
                parts.push_back({P->src_lo, P->src_lo + main_n, spl});
            }
        }
        if (parts.empty())
            for (int64_t lo = P->src_lo; lo < P->src_hi; lo += sb) parts.push_back({lo, std::min<int64_t>(P->src_hi, lo + sb), spl});
        const bool concurrent = parts.size() == 2 && single;
        cudaStream_t st2 = concurrent ? side_stream(P->device) : st;
        cudaEvent_t ev_in = nullptr, ev_out = nullptr;
        if (concurrent) {
            WR_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
            WR_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
        }
        struct PartBufs {
            DBuf<uint32_t> rows;
            DBuf<int> tile_src, slot_row, pos_of, flat, done_list, fuse_ctr;
            BfRun run;
            int ntiles = 0, tsw = 0;
        };
        std::vector<PartBufs> pb(concurrent ? 2 : 1);
        auto prepare = [&](PartBufs &b, const Part &pt, int64_t cap_tiles) {
            b.tsw = 32 * pt.spl * pk;
            if (!b.rows.p) {
                b.rows.alloc((size_t)cap_tiles * V * 32 * pt.spl);
                b.tile_src.alloc(cap_tiles * b.tsw);
                b.slot_row.alloc(cap_tiles * b.tsw);
                b.pos_of.alloc(concurrent ? pt.hi - pt.lo : sb);
                b.flat.alloc(o.pred_out ? cap_tiles : 0);
                b.done_list.alloc(fused ? cap_tiles : 0);
                b.fuse_ctr.alloc(fused ? 4 : 0);
            }
            b.ntiles = make_tiles_ordered(g, P->sources.p, pt.lo, pt.hi, b.tsw, cap_tiles, b.tile_src.p,
                                          b.slot_row.p, b.pos_of.p, st);
            b.run = BfRun{b.tile_src.p, b.ntiles, b.rows.p, WR_BF_FRONTIER, max_rounds, pt.spl, b.slot_row.p};
            b.run.pack = pk;
            b.run.keyed = pk == 2 && keyed;
            b.run.nf_delta = (pk == 1 && (o.flags & WR_ROUTE_NEARFAR)) ? nf_delta_for(g) : 0.f;
            b.run.ovf_thr = pk != 2 ? 0u
                            : b.run.keyed ? (0x7ffu - (uint32_t)g->max_abs_w) << 4
                                          : 0x7fffu - (uint32_t)g->max_abs_w;
            if (fused) {
                WR_CUDA(cudaMemsetAsync(b.flat.p, 0, sizeof(int) * b.ntiles, st));
                WR_CUDA(cudaMemsetAsync(b.done_list.p, 0xff, sizeof(int) * b.ntiles, st));
                WR_CUDA(cudaMemsetAsync(b.fuse_ctr.p, 0, sizeof(int) * 4, st));
                b.run.fuse.pred_out = o.pred_out;
                b.run.fuse.out_row0 = pt.lo - P->src_lo;
                b.run.fuse.flat_tiles = b.flat.p;
                b.run.fuse.done_list = b.done_list.p;
                b.run.fuse.counters = b.fuse_ctr.p;
            }
            tiles_swept += b.ntiles;
            tile_width = std::max(tile_width, b.tsw);
        };
        auto gather = [&](PartBufs &b, const Part &pt, cudaStream_t s_) {
            if (P->B <= 0) return;
            gather_send_kernel<<<gridn(P->B * WR_MAX_STOPS, 256), 256, 0, s_>>>(
                P->stops.p, P->n_arr.p, P->status.p, P->B, P->src_row.p, P->src_lo, P->src_hi, pt.lo, pt.hi, off_r,
                b.rows.p, V, b.tsw, b.run.keyed ? 3 : pk, b.pos_of.p, (uint32_t *)send);
            count_launch();
            WR_LAUNCH_CHECK();
        };
        for (size_t ip = 0; ip < parts.size(); ++ip) {
            if (concurrent && ip == 1) break;   // both parts run below
            const Part &pt = parts[ip];
            PartBufs &b = pb[0];
            if (concurrent) {
                prepare(pb[0], parts[0], (parts[0].hi - parts[0].lo + 32LL * parts[0].spl * pk - 1) /
                                             (32LL * parts[0].spl * pk));
                prepare(pb[1], parts[1], (parts[1].hi - parts[1].lo) / (32LL * parts[1].spl * pk));
            } else {
                prepare(b, pt, max_tiles);
            }
            WR_CUDA(cudaEventRecord(b0, st));
            const double host_to_b0 =
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hclock0).count();
            if (concurrent) {
                WR_CUDA(cudaEventRecord(ev_in, st));
                WR_CUDA(cudaStreamWaitEvent(st2, ev_in, 0));
                {
                    StreamScope side(st2);   // the tail's temporaries live in st2's order
                    NvtxRange nv("wr.bf.sweep+pred (tail)");
                    bf_run(g, pb[0].run, d_stats.p, st2);
                    gather(pb[0], parts[0], st2);
                }
                {
                    NvtxRange nv(fused ? "wr.bf.sweep+pred" : "wr.bf.sweep");
                    bf_run(g, pb[1].run, d_stats.p, st);
                }
                WR_CUDA(cudaEventRecord(ev_out, st2));
                WR_CUDA(cudaStreamWaitEvent(st, ev_out, 0));   // every later free on st follows the tail
            } else {
                NvtxRange nv(fused ? "wr.bf.sweep+pred" : "wr.bf.sweep");
                bf_run(g, b.run, d_stats.p, st);
            }
            WR_CUDA(cudaEventRecord(b1, st));
            if (o.pred_out && !concurrent) {   // a4 canonical pred of this segment's sources
                if (!fused) {
                    WR_CUDA(cudaMemsetAsync(b.flat.p, 0, sizeof(int) * b.ntiles, st));
                    bf_write_outputs(g, b.run, pt.lo - P->src_lo, P->S, nullptr, V, nullptr, o.pred_out, b.flat.p, st);
                }
                std::vector<int> hflat(b.ntiles);
                WR_CUDA(cudaMemcpyAsync(hflat.data(), b.flat.p, sizeof(int) * b.ntiles, cudaMemcpyDeviceToHost, st));
                WR_CUDA(cudaStreamSynchronize(st));
                std::vector<int> todo;
                for (int t = 0; t < b.ntiles; ++t)
                    if (hflat[t] || g->has_negative) todo.push_back(t);
                // packed rows: w > 0 admits no flat vertex unless a distance
                // was clipped, and then the overflow flag forces the redo
                if (pk == 2) todo.clear();
                bf_resolve_flat(g, b.run, todo, pt.lo - P->src_lo, o.pred_out, st);
            }
            WR_CUDA(cudaEventRecord(b2, st));
            WR_CUDA(cudaEventSynchronize(b2));
            float x = 0.f, y = 0.f;
            WR_CUDA(cudaEventElapsedTime(&x, b0, b1));
            WR_CUDA(cudaEventElapsedTime(&y, b1, b2));
            bf_ms += x;
            pred_ms += y;
            if (concurrent) gather(pb[1], parts[1], st);
            else gather(b, pt, st);
            ++segments;
            if (trace) {
                WR_CUDA(cudaEventRecord(t1, st));
                WR_CUDA(cudaEventSynchronize(t1));
                float a = 0.f, c = 0.f;
                WR_CUDA(cudaEventElapsedTime(&a, t0, b0));
                WR_CUDA(cudaEventElapsedTime(&c, b2, t1));
                fprintf(stderr,
                        "[wr] local segment %d (%d tiles%s): alloc+tiles %.2f ms device (%.2f ms host), "
                        "gather_send %.2f ms; host: prologue %.2f, budget %.2f\n",
                        segments, concurrent ? pb[0].ntiles + pb[1].ntiles : b.ntiles,
                        concurrent ? ", wide + concurrent narrow tail" : "", a, host_to_b0, c, h_pre,
                        h_budget - h_pre);
            }
        }
        if (concurrent) {
            cudaEventDestroy(ev_in);
            cudaEventDestroy(ev_out);
        }
        if (trace) {
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
        }
        cudaEventDestroy(b0);
        cudaEventDestroy(b1);
        cudaEventDestroy(b2);
    };
    run_phase(pack);
    WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    if (pack == 2 && keyed && hs.overflow) {   // a distance may not fit in 11 bits: plain packed rows
        const BfTileStats z{0ull, 0, -1, 0ull};
        WR_CUDA(cudaMemcpyAsync(d_stats.p, &z, sizeof(z), cudaMemcpyHostToDevice, st));
        keyed = false;
        tiles_swept = 0;
        run_phase(2);
        WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
    }
    if (pack == 2 && hs.overflow) {   // a distance may not fit in 15 bits: redo with 32-bit rows
        const BfTileStats z{0ull, 0, -1, 0ull};
        WR_CUDA(cudaMemcpyAsync(d_stats.p, &z, sizeof(z), cudaMemcpyHostToDevice, st));
        pack = 1;
        tiles_swept = 0;
        run_phase(1);
    }
    const double h_loop = hms();
    WR_CUDA(cudaEventRecord(e1, st));
    WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    static const bool trace_l = getenv("WR_TRACE") != nullptr;
    if (trace_l) fprintf(stderr, "[wr] local host: loop done at %.2f ms, synced at %.2f ms\n", h_loop, hms());
    float ms = 0.f;
    WR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (hs.negcycle_tile >= 0) return fail(WR_ENEGCYCLE, "wr_orders_local: negative cycle reachable");
    if (stats) {
        stats->sources = nsrc;
        stats->segments = segments;
        stats->rounds_max = hs.rounds_max;
        stats->relaxations = (int64_t)hs.relax;
        stats->visits = (int64_t)hs.visits;
        stats->ms = ms;
        stats->kernel_launches = g_launches - l0;
        stats->bf_ms = bf_ms;
        stats->pred_ms = pred_ms;
        stats->row_bits = pack == 2 ? 16 : 32;
        stats->keyed = pack == 2 && keyed ? 1 : 0;
        stats->tiles = tiles_swept;
        stats->tile_sources = tile_width;
    }
    return WR_OK;
}

template <class C>
static void route_block(const Plan &P, const uint32_t *Dall, int64_t o_lo, int64_t nord, wr_route_result *d_res,
                        unsigned long long *d_counters, cudaStream_t st) {
    if (nord <= 0) return;
    NvtxRange nv("wr.routes");
    const int *xy = P.g->xy.p;
    DBuf<OrderRoute> ordr(nord);
    DBuf<int> pcnt(nord + 1), icnt(nord + 1), hk_ctr(8), hk_list(nord), shk_list(nord);
    WR_CUDA(cudaMemsetAsync(pcnt.p + nord, 0, 4, st));
    WR_CUDA(cudaMemsetAsync(icnt.p + nord, 0, 4, st));
    WR_CUDA(cudaMemsetAsync(hk_ctr.p, 0, 32, st));
    route_prepare_kernel<C><<<gridn(nord, 128), 128, 0, st>>>(
        P.n_arr.p, P.status.p, P.stops.p, o_lo, nord, Dall, P.m, xy,
        P.labels.p ? P.labels.p + o_lo * WR_MAX_STOPS : nullptr, P.chunk, ordr.p, pcnt.p, icnt.p, P.pairs,
        hk_ctr.p, hk_list.p, P.closed ? P.dep_info.p : nullptr, shk_list.p);
    count_launch();
    WR_LAUNCH_CHECK();
    scan_exclusive_i32(pcnt.p, pcnt.p, (int)(nord + 1), st);
    scan_exclusive_i32(icnt.p, icnt.p, (int)(nord + 1), st);
    int nprob = 0, nitems = 0, hkc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    WR_CUDA(cudaMemcpyAsync(&nprob, pcnt.p + nord, 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaMemcpyAsync(&nitems, icnt.p + nord, 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaMemcpyAsync(hkc, hk_ctr.p, 32, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    const int nhk = hkc[0];
    DBuf<RouteProblem> probs(std::max(nprob, 1));
    DBuf<RouteWorkItem> items(std::max(nitems, 1));
    DBuf<uint64_t> item_best(std::max(nitems, 1)), prob_best(std::max(nprob, 1));
    route_emit_kernel<<<gridn(nord, 128), 128, 0, st>>>(nord, ordr.p, pcnt.p, icnt.p, P.chunk, probs.p, items.p);
    count_launch();
    WR_LAUNCH_CHECK();
    if (nitems > 0) {
        // measured: replicated copies halve an 11-stop exact batch (C4 m = 1:
        // 164 -> 82 ms/step) but cost ~2 ms on C5's 6-8-stop orders (lower
        // occupancy), so they serve launches whose largest problem has >= 9
        const int ns_max = std::max(2, hkc[3]);
        const bool rep = ns_max >= 9;
        const size_t esmem = (size_t)ENUM_WARPS * ns_max * ns_max * (rep ? 32 : 1) * sizeof(uint32_t);
        if (rep) {
            WR_CUDA(cudaFuncSetAttribute(route_enum_kernel<C, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)esmem));
            route_enum_kernel<C, 5><<<gridn(nitems, ENUM_WARPS), ENUM_WARPS * 32, esmem, st>>>(
                probs.p, items.p, nitems, Dall, item_best.p, ns_max);
        } else {
            route_enum_kernel<C, 0><<<gridn(nitems, ENUM_WARPS), ENUM_WARPS * 32, esmem, st>>>(
                probs.p, items.p, nitems, Dall, item_best.p, ns_max);
        }
        problem_reduce_kernel<<<gridn(nprob, 128), 128, 0, st>>>(probs.p, nprob, item_best.p, prob_best.p);
        count_launch();
        count_launch();
        WR_LAUNCH_CHECK();
    }
    route_finalize_kernel<C><<<gridn(nord, 4), 128, 0, st>>>(nord, ordr.p, prob_best.p, probs.p, Dall, P.stops.p,
                                                             o_lo, d_res, d_counters, P.pairs);
    count_launch();
    WR_LAUNCH_CHECK();
    if (P.pairs) {
        route_pairs_kernel<C><<<(unsigned)nord, PAIRS_THREADS, 0, st>>>(nord, ordr.p, Dall, P.stops.p, o_lo, d_res,
                                                                      d_counters);
        count_launch();
        WR_LAUNCH_CHECK();
    }
    if (hkc[4] > 0) {   // 8-stop exact routes: warp Held-Karp
        static bool attr = false;
        if (!attr) {
            WR_CUDA(cudaFuncSetAttribute(route_hk_small_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SHK_SMEM));
            attr = true;
        }
        route_hk_small_kernel<C><<<gridn(hkc[4], SHK_WARPS), SHK_WARPS * 32, SHK_SMEM, st>>>(
            shk_list.p, hkc[4], ordr.p, Dall, P.stops.p, o_lo, d_res, d_counters, hk_lists(P.device));
        count_launch();
        WR_LAUNCH_CHECK();
    }
    if (nhk > 0) {   // 13-16-stop exact routes: one order per 8-CTA cluster, L2-resident tables
        const int nmax = hkc[2];
        const int ncl = std::min(nhk, HK_CLUSTERS);
        const size_t stride = ((size_t)1 << nmax) * HK_RS;
        DBuf<uint32_t> ws((size_t)ncl * stride);
        route_hk_kernel<C><<<ncl * HK_CL, HK_THREADS, 0, st>>>(hk_list.p, nhk, ordr.p, Dall, P.stops.p, o_lo, d_res,
                                                               d_counters, hk_ctr.p + 1, ws.p, stride,
                                                               hk_lists(P.device));
        count_launch();
        WR_LAUNCH_CHECK();
        WR_CUDA(cudaStreamSynchronize(st));   // workspace lifetime
    }
    WR_CUDA(cudaStreamSynchronize(st));   // temporaries are freed on return
}

static wr_status finish_impl(wr_plan *P, const void *gathered, wr_route_result *results, const wr_route_opts *opts,
                             wr_route_stats *stats) {
    if (!P) return fail(WR_EINVAL, "wr_orders_finish: null plan");
    const int64_t nord = P->order_hi - P->order_lo;
    if (nord > 0 && !results) return fail(WR_EINVAL, "wr_orders_finish: results");
    if (nord > 0 && !is_device_ptr(gathered)) return fail(WR_EINVAL, "wr_orders_finish: gathered must be device memory");
    WR_CUDA(cudaSetDevice(P->device));
    const int64_t l0 = g_launches;
    wr_route_opts o{};
    if (opts) o = *opts;
    cudaStream_t st = (cudaStream_t)o.stream;
    StreamScope stream_scope(st);
    cudaEvent_t e0, e1;
    WR_CUDA(cudaEventCreate(&e0));
    WR_CUDA(cudaEventCreate(&e1));
    WR_CUDA(cudaEventRecord(e0, st));
    DBuf<unsigned long long> counters(2);
    WR_CUDA(cudaMemsetAsync(counters.p, 0, 16, st));
    const bool res_dev = is_device_ptr(results);
    DBuf<wr_route_result> d_res;
    wr_route_result *dres = (wr_route_result *)results;
    if (nord > 0) {
        DBuf<uint32_t> Dall((size_t)nord * DSTRIDE);
        WR_CUDA(cudaMemsetAsync(Dall.p, 0, Dall.bytes(), st));
        assemble_kernel<<<gridn(nord * WR_MAX_STOPS, 256), 256, 0, st>>>(
            P->stops.p, P->n_arr.p, P->status.p, P->B, P->order_lo, P->order_hi, P->src_row.p, P->blk.p, P->world,
            P->off_all.p, (const uint32_t *)gathered, P->max_send, Dall.p);
        count_launch();
        WR_LAUNCH_CHECK();
        if (!res_dev) {
            d_res.alloc(nord);
            dres = d_res.p;
        }
        if (P->g->wtype == WR_F32) route_block<CostF32>(*P, Dall.p, P->order_lo, nord, dres, counters.p, st);
        else route_block<CostI32>(*P, Dall.p, P->order_lo, nord, dres, counters.p, st);
        if (!res_dev)
            WR_CUDA(cudaMemcpyAsync(results, d_res.p, sizeof(wr_route_result) * nord, cudaMemcpyDeviceToHost, st));
    }
    WR_CUDA(cudaEventRecord(e1, st));
    unsigned long long hc[2] = {0, 0};
    WR_CUDA(cudaMemcpyAsync(hc, counters.p, 16, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    WR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats) {
        stats->orders = nord;
        stats->permutations = (int64_t)hc[0];
        stats->stitch_candidates = (int64_t)hc[1];
        stats->ms = ms;
        stats->kernel_launches = g_launches - l0;
    }
    return WR_OK;
}

// int32 route sums must stay exact: (n-1) legs of at most (V-1)*max|w|.
static wr_status check_route_overflow(const wr_graph *g) {
    if (g->wtype == WR_I32 &&
        (int64_t)(WR_MAX_STOPS - 1) * (int64_t)(g->V - 1) * (int64_t)g->max_abs_w >= (int64_t)INT32_MAX)
        return fail(WR_EOVERFLOW, "route: (15)(V-1)max|w| >= INT32_MAX, int32 route sums could overflow");
    return WR_OK;
}

int ctx_rank(const wr_ctx *c);
int ctx_world(const wr_ctx *c);
void ctx_allgather(const wr_ctx *c, const void *send, void *recv, size_t bytes, cudaStream_t st);
void ctx_share_blocks(const wr_ctx *c, void *buf, const int64_t *off, cudaStream_t st);

static wr_status route_orders_impl(const wr_graph *g, const int64_t *order_ptr, const int32_t *order_nodes,
                                   int64_t B, const wr_route_opts *opts, const int32_t *labels16,
                                   const int32_t *line_labels, wr_route_result *results, wr_route_stats *stats) {
    if (!g) return fail(WR_EINVAL, "wr_route_orders: null graph");
    if (wr_status r = check_route_overflow(g)) return r;
    WR_CUDA(cudaSetDevice(g->device));
    const int64_t l0 = g_launches;
    wr_route_opts o{};
    if (opts) o = *opts;
    cudaStream_t st = (cudaStream_t)o.stream;
    StreamScope stream_scope(st);
    cudaEvent_t e0, e1;
    WR_CUDA(cudaEventCreate(&e0));
    WR_CUDA(cudaEventCreate(&e1));
    WR_CUDA(cudaEventRecord(e0, st));
    const wr_ctx *ctx = o.ctx;
    const int rank = ctx_rank(ctx), world = ctx_world(ctx);
    if (B > 0 && !results) return fail(WR_EINVAL, "wr_route_orders: results");
    wr_plan *P = nullptr;
    wr_status rc = plan_impl(g, order_ptr, order_nodes, B, rank, world, &o, labels16, line_labels, &P);
    if (rc) return rc;
    std::unique_ptr<wr_plan> hold(P);
    DBuf<uint32_t> send(std::max<int64_t>(P->max_send, 1));
    wr_route_stats s1{}, s2{};
    rc = local_impl(P, send.p, &o, &s1);
    if (rc) return rc;
    if (!ctx) {
        rc = finish_impl(P, send.p, results, &o, &s2);
        if (rc) return rc;
    } else {
        // a9: ONE all-gather of the owned D entries (rank-major, max_send
        // 32-bit words each), then this rank's order block, then (unless
        // WR_ROUTE_RANK_RESULTS) the result blocks of every rank
        DBuf<uint32_t> gathered((size_t)world * P->max_send);
        ctx_allgather(ctx, send.p, gathered.p, (size_t)P->max_send * 4, st);
        const bool res_dev = is_device_ptr(results);
        const bool share = !(o.flags & WR_ROUTE_RANK_RESULTS) && world > 1;
        DBuf<wr_route_result> dres;
        wr_route_result *full = results;
        if (!res_dev && share) {
            dres.alloc(std::max<int64_t>(B, 1));
            full = dres.p;
        }
        rc = finish_impl(P, gathered.p, full + P->order_lo, &o, &s2);
        if (rc) return rc;
        if (share) {
            std::vector<int64_t> off(world + 1);
            for (int q = 0; q < world; ++q) {
                int64_t lo, hi;
                wr_shard_range(B, q, world, &lo, &hi);
                off[q] = lo * (int64_t)sizeof(wr_route_result);
                off[q + 1] = hi * (int64_t)sizeof(wr_route_result);
            }
            ctx_share_blocks(ctx, full, off.data(), st);
            if (!res_dev)
                WR_CUDA(cudaMemcpyAsync(results, full, sizeof(wr_route_result) * B, cudaMemcpyDeviceToHost, st));
        }
    }
    WR_CUDA(cudaEventRecord(e1, st));
    WR_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    WR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    static const bool trace = getenv("WR_TRACE") != nullptr;
    if (trace)
        fprintf(stderr, "[wr] route_orders %.2f ms: local %.2f (bf %.2f, pred %.2f), finish %.2f, plan+rest %.2f\n", ms,
                s1.ms, s1.bf_ms, s1.pred_ms, s2.ms, ms - s1.ms - s2.ms);
    if (stats) {
        *stats = s2;
        stats->orders = B;
        stats->sources = P->S;
        stats->segments = s1.segments;
        stats->rounds_max = s1.rounds_max;
        stats->relaxations = s1.relaxations;
        stats->visits = s1.visits;
        stats->ms = ms;
        stats->kernel_launches = g_launches - l0;
        stats->bf_ms = s1.bf_ms;
        stats->pred_ms = s1.pred_ms;
        stats->row_bits = s1.row_bits;
        stats->keyed = s1.keyed;
        stats->tiles = s1.tiles;
        stats->tile_sources = s1.tile_sources;
    }
    return WR_OK;
}

}  // namespace wr

extern "C" {

wr_status wr_orders_plan(const wr_graph *g, const int64_t *order_ptr, const int32_t *order_nodes, int64_t B,
                         const int32_t *labels, int32_t rank, int32_t world, const wr_route_opts *opts,
                         wr_plan **out) {
    return wr::guarded([&] {
        wr::NvtxRange nv("wr_orders_plan");
        if (wr_status r = g ? wr::check_route_overflow(g) : WR_OK) return r;
        return wr::plan_impl(g, order_ptr, order_nodes, B, rank, world, opts, nullptr, labels, out);
    });
}

wr_status wr_plan_info(const wr_plan *p, wr_plan_info_t *info) {
    if (!p || !info) return wr::fail(WR_EINVAL, "wr_plan_info: null argument");
    info->B = p->B;
    info->S = p->S;
    info->rank = p->rank;
    info->world = p->world;
    info->src_lo = p->src_lo;
    info->src_hi = p->src_hi;
    info->order_lo = p->order_lo;
    info->order_hi = p->order_hi;
    info->send_count = p->send_count;
    info->max_send = p->max_send;
    info->wtype = p->g->wtype;
    return WR_OK;
}

wr_status wr_orders_local(wr_plan *p, void *send, const wr_route_opts *opts, wr_route_stats *stats) {
    return wr::guarded([&] {
        wr::NvtxRange nv("wr_orders_local");
        return wr::local_impl(p, send, opts, stats);
    });
}

wr_status wr_orders_finish(wr_plan *p, const void *gathered, wr_route_result *results, const wr_route_opts *opts,
                           wr_route_stats *stats) {
    return wr::guarded([&] {
        wr::NvtxRange nv("wr_orders_finish");
        return wr::finish_impl(p, gathered, results, opts, stats);
    });
}

wr_status wr_plan_free(wr_plan *p) {
    if (!p) return WR_OK;
    return wr::guarded([&] {
        WR_CUDA(cudaSetDevice(p->device));
        delete p;
        return WR_OK;
    });
}

wr_status wr_route_orders(const wr_graph *g, const int64_t *order_ptr, const int32_t *order_nodes, int64_t B,
                          const int32_t *labels, const wr_route_opts *opts, wr_route_result *results,
                          wr_route_stats *stats) {
    return wr::guarded([&] {
        wr::NvtxRange nv("wr_route_orders");
        return wr::route_orders_impl(g, order_ptr, order_nodes, B, opts, nullptr, labels, results, stats);
    });
}

wr_status wr_route_segmented(const wr_graph *g, const int32_t *stops, int32_t n, const int32_t *labels, int32_t m,
                             const wr_route_opts *opts, wr_route_result *out) {
    return wr::guarded([&]() -> wr_status {
        if (!g || !out || n < 0 || (n > 0 && !stops)) return wr::fail(WR_EINVAL, "wr_route_segmented: bad arguments");
        if (n > WR_MAX_STOPS) return wr::fail(WR_ETOOLARGE, "wr_route_segmented: n > 16");
        std::vector<int32_t> hs(n);
        if (n) WR_CUDA(cudaMemcpy(hs.data(), stops, 4LL * n, cudaMemcpyDefault));
        std::vector<int32_t> uniq(hs);
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        std::vector<int32_t> lab16(WR_MAX_STOPS, 0);
        if (labels) {
            std::vector<int32_t> hl(uniq.size());
            if (!uniq.empty()) WR_CUDA(cudaMemcpy(hl.data(), labels, 4 * uniq.size(), cudaMemcpyDefault));
            for (size_t i = 0; i < uniq.size(); ++i) lab16[i] = hl[i];
        }
        int64_t ptr[2] = {0, n};
        wr_route_opts o{};
        if (opts) o = *opts;
        o.m = m;
        if (labels && m < 2) o.m = 2;   // caller labels always go through the stitch
        o.ctx = nullptr;
        o.flags &= ~WR_ROUTE_CLOSED;   // one stop set, open route (closed tours: wr_route_orders)
        return wr::route_orders_impl(g, ptr, hs.data(), 1, &o, labels ? lab16.data() : nullptr, nullptr, out, nullptr);
    });
}

wr_status wr_segment_plan(const int32_t *xy, int32_t n, int32_t m, int32_t *labels_out, int32_t device) {
    return wr::guarded([&]() -> wr_status {
        if (!xy || !labels_out || n < 1 || n > WR_MAX_STOPS || m < 1)
            return wr::fail(WR_EINVAL, "wr_segment_plan: bad arguments (1 <= n <= 16, m >= 1)");
        WR_CUDA(cudaSetDevice(device));
        std::vector<int32_t> h(2 * n);
        WR_CUDA(cudaMemcpy(h.data(), xy, 8LL * n, cudaMemcpyDefault));
        for (int v : h)
            if (v <= -(1 << 20) || v >= (1 << 20)) return wr::fail(WR_EINVAL, "wr_segment_plan: |xy| >= 2^20");
        wr::DBuf<int> dxy = wr::to_device<int>(h.data(), 2 * n, 0), dl(n);
        wr::segment_plan_kernel<<<1, 32>>>(dxy.p, n, m, dl.p);
        wr::count_launch();
        WR_LAUNCH_CHECK();
        WR_CUDA(cudaMemcpy(labels_out, dl.p, 4LL * n, cudaMemcpyDefault));
        return WR_OK;
    });
}

wr_status wr_route_cost(int32_t wtype, const void *D, int32_t n, const int32_t *seqs, int32_t len, int64_t count,
                        void *costs, void *stream) {
    return wr::guarded([&]() -> wr_status {
        if ((wtype != WR_I32 && wtype != WR_F32) || n < 1 || !D || len < 0 || count < 0 ||
            (count > 0 && (!seqs || !costs)))
            return wr::fail(WR_EINVAL, "wr_route_cost: bad arguments");
        if (count == 0) return WR_OK;
        cudaStream_t st = (cudaStream_t)stream;
        wr::StreamScope stream_scope(st);
        int dev = 0;
        WR_CUDA(cudaGetDevice(&dev));
        wr::DBuf<uint32_t> dD = wr::to_device<uint32_t>((const uint32_t *)D, (size_t)n * n, st);
        wr::DBuf<int> dS = wr::to_device<int>(seqs, (size_t)count * len, st);
        const bool cdev = wr::is_device_ptr(costs);
        wr::DBuf<uint32_t> dC;
        uint32_t *cp = (uint32_t *)costs;
        if (!cdev) {
            dC.alloc(count);
            cp = dC.p;
        }
        wr::DBuf<int> bad(1);
        WR_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
        if (wtype == WR_F32)
            wr::route_cost_kernel<wr::CostF32><<<wr::gridn(count, 256), 256, 0, st>>>(dD.p, n, dS.p, len, count, cp, bad.p);
        else
            wr::route_cost_kernel<wr::CostI32><<<wr::gridn(count, 256), 256, 0, st>>>(dD.p, n, dS.p, len, count, cp, bad.p);
        wr::count_launch();
        WR_LAUNCH_CHECK();
        int hb = 0;
        WR_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, st));
        if (!cdev) WR_CUDA(cudaMemcpyAsync(costs, dC.p, 4 * count, cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
        if (hb & 1) return wr::fail(WR_EINVAL, "wr_route_cost: sequence index outside [0, n)");
        if (hb & 2) return wr::fail(WR_EOVERFLOW, "wr_route_cost: int32 route sum overflows");
        return WR_OK;
    });
}

}  // extern "C"
