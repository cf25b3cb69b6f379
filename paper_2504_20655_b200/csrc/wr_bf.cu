// wr_bf.cu - a3 batched Bellman-Ford relaxation sweep, a4 canonical
// predecessor, a8 source-batch scheduler, and the wr_bf_batch entry point.
//
// The paper's kernel (P720-724 §4.7) is edge-parallel, one thread per edge,
// (V-1) rounds with a host sync per round, dist/pred V x N in global memory
// with write contention. This design is B200-first instead:
//   * sources are the SIMD lanes: a tile of 32*SPL sources stores one
//     128*SPL-byte row per vertex (rows[tile][v][slot]); lane l owns the SPL
//     consecutive slots l*SPL.., so every neighbour gather is a fully
//     coalesced vector load and each graph arc (u, w) is fetched once per
//     32*SPL relaxations;
//   * one CTA owns a tile and iterates its rounds alone (no grid sync, no
//     host sync per round - the paper's 10.3 us/round), tiles are claimed
//     from a persistent work counter;
//   * frontier pull: a round relaxes only vertices with an in-neighbour that
//     improved in the previous round (two V-bit bitmaps in shared memory);
//     the improvement of a vertex is one __any_sync vote, and the improving
//     warp marks its out-neighbours for the next round lane-parallel;
//   * atomic-free commit: each (v, slot) has exactly one writer (the warp
//     that owns v's candidate word), updates are in place (chaotic /
//     Gauss-Seidel), which reaches the same unique fixpoint (reading O2:
//     the relaxation operator is monotone and deflationary for w >= 0, and
//     exact for int weights), so dist is bit-identical to the oracle;
//   * pred is not written inside the racy sweep: a4 recomputes the
//     canonical predecessor from the converged dist (O3), deterministic.
#include <algorithm>
#include <cmath>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <type_traits>
#include <string>
#include <vector>

#include "wr_internal.cuh"

namespace wr {

constexpr uint32_t FULL = 0xffffffffu;

// ------------------------------------------------------------- weight ops --
// Nonnegative int32: unsigned add + min (DPX VIADDMNMX). INF = INT32_MAX, and
// INF + w (w < 2^31) never wraps and never beats a finite value: an INF tail
// relaxes nothing, exactly like the oracle's "skip d[u] == INF".
struct OpU32 {
    static constexpr int PACK = 1;   // sources per 32-bit word
    static constexpr bool KEYED = false;
    __device__ __forceinline__ static uint32_t prep_w(uint32_t w, int) { return w; }
    __device__ __forceinline__ static uint32_t min_word(uint32_t a, uint32_t b) { return less(a, b) ? a : b; }
    __device__ __forceinline__ static bool any_less(uint32_t a, uint32_t b) { return less(a, b); }
    __device__ __forceinline__ static bool overflow(uint32_t, uint32_t) { return false; }
    __device__ __forceinline__ static uint32_t half(uint32_t x, int) { return x; }
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
    // tight and d[u] < d[v], for a finite dv: w > 0 and du + w == dv (an INF
    // du gives du + w > INF > dv, no wrap for w < 2^31)
    __device__ __forceinline__ static bool steep_tight(uint32_t du, uint32_t w, uint32_t dv) {
        return w != 0u && du + w == dv;
    }
};
// fp32 (weights finite, >= 0): one IEEE binary32 RN add, then min. +inf
// tails give +inf, which never wins.
struct OpF32 {
    static constexpr int PACK = 1;   // sources per 32-bit word
    static constexpr bool KEYED = false;
    __device__ __forceinline__ static uint32_t prep_w(uint32_t w, int) { return w; }
    __device__ __forceinline__ static uint32_t min_word(uint32_t a, uint32_t b) { return less(a, b) ? a : b; }
    __device__ __forceinline__ static bool any_less(uint32_t a, uint32_t b) { return less(a, b); }
    __device__ __forceinline__ static bool overflow(uint32_t, uint32_t) { return false; }
    __device__ __forceinline__ static uint32_t half(uint32_t x, int) { return x; }
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
    __device__ __forceinline__ static bool steep_tight(uint32_t du, uint32_t w, uint32_t dv) {
        return tight(du, w, dv) && less(du, dv);
    }
};
// int32 with negative weights: exact 64-bit candidate, INF tails skipped.
struct OpI32N {
    static constexpr int PACK = 1;   // sources per 32-bit word
    static constexpr bool KEYED = false;
    __device__ __forceinline__ static uint32_t prep_w(uint32_t w, int) { return w; }
    __device__ __forceinline__ static uint32_t min_word(uint32_t a, uint32_t b) { return less(a, b) ? a : b; }
    __device__ __forceinline__ static bool any_less(uint32_t a, uint32_t b) { return less(a, b); }
    __device__ __forceinline__ static bool overflow(uint32_t, uint32_t) { return false; }
    __device__ __forceinline__ static uint32_t half(uint32_t x, int) { return x; }
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
    __device__ __forceinline__ static bool steep_tight(uint32_t du, uint32_t w, uint32_t dv) {
        return tight(du, w, dv) && less(du, dv);
    }
};
// Nonnegative int32 distances that provably stay below 2^15 - 1, two per
// 32-bit word (packed u16, DPX VIADDMNMX.U16x2: two relaxations per
// instruction, half the bytes per source row). INF = 0x7fff per half; with
// w clamped to <= 0x7fff, du + w <= 0xfffe never wraps and an INF tail
// never beats a finite value. A path longer than 0x7ffe cannot be
// represented: the sweep flags a tile whose stored distances reach
// 0x7fff - max_w (any longer candidate could be clipped) and the caller
// redoes the segment with 32-bit rows, so results are exact either way.
struct OpU16 {
    static constexpr int PACK = 2;
    static constexpr bool KEYED = false;
    static constexpr uint32_t INF = 0x7fff7fffu;
    static constexpr uint32_t INF1 = 0x7fffu;
    static constexpr uint32_t ZERO = 0u;
    static constexpr uint16_t SEED16 = 0;
    __device__ __forceinline__ static uint32_t prep_w(uint32_t w, int) {
        w = min(w, 0x7fffu);
        return w | (w << 16);
    }
    __device__ __forceinline__ static uint32_t relax(uint32_t d, uint32_t du, uint32_t w2) {
        return __viaddmin_u16x2(du, w2, d);
    }
    __device__ __forceinline__ static uint32_t min_word(uint32_t a, uint32_t b) { return __vminu2(a, b); }
    __device__ __forceinline__ static bool any_less(uint32_t a, uint32_t b) { return __vcmpltu2(a, b) != 0u; }
    __device__ __forceinline__ static bool overflow(uint32_t d, uint32_t thr2) {
        return (__vcmpgeu2(d, thr2) & ~__vcmpeq2(d, INF)) != 0u;
    }
    __device__ __forceinline__ static uint32_t half(uint32_t x, int h) { return (x >> (16 * h)) & 0xffffu; }
    // per-slot (one half) predicates for the pred pass
    __device__ __forceinline__ static bool finite(uint32_t x1) { return x1 != INF1; }
    __device__ __forceinline__ static bool steep_tight(uint32_t du1, uint32_t w, uint32_t dv1) {
        return w != 0u && du1 + w == dv1;   // w > 0 on every packed graph
    }
};

// Keyed packed rows (the routing path with fused pred): each u16 half holds
// key = d << 4 | k, where k is the in-arc index (in v's CSC range, sorted by
// tail) of the arc that set d - the canonical pred (O3: the smallest steep
// tight tail; with every weight >= 1 each tight arc is steep) rides along
// with the distance, so the pred pass only decodes k instead of re-testing
// every in-arc of every vertex against the final distances. One add-min
// per relaxation relaxes both: c = (x | 0xf) + ((w << 4) + k - 15) strips
// the tail's own k and appends this arc's, and min over keys is min over
// d, ties -> smallest k (smallest tail). Every tight arc is offered to v
// after its tail's last change (delta pull), so the final key holds the
// smallest tight k whatever the schedule (min is order-free). k = 15 is
// NONE: the seed key 0x000f (d = 0, source) and INF 0x7fff (unreachable)
// decode to pred -1. Needs in-degree <= 15, w in [1, 0x7ff], d < 0x7ff
// (a stored distance reaching 0x7ff - max_w raises the overflow flag and
// the phase is redone with plain packed, then 32-bit rows).
struct OpK16 {
    static constexpr int PACK = 2;
    static constexpr bool KEYED = true;
    static constexpr uint32_t INF = 0x7fff7fffu;
    static constexpr uint32_t INF1 = 0x7fffu;
    static constexpr uint32_t ZERO = 0x000f000fu;
    static constexpr uint16_t SEED16 = 0x000f;
    __device__ __forceinline__ static uint32_t prep_w(uint32_t w, int k) {
        const uint32_t x = (min(w, 0x7ffu) << 4) + (uint32_t)k - 15u;   // w >= 1: x >= 1
        return x | (x << 16);
    }
    __device__ __forceinline__ static uint32_t relax(uint32_t d, uint32_t du, uint32_t w2) {
        return __viaddmin_u16x2(du | 0x000f000fu, w2, d);
    }
    __device__ __forceinline__ static uint32_t min_word(uint32_t a, uint32_t b) { return __vminu2(a, b); }
    __device__ __forceinline__ static bool any_less(uint32_t a, uint32_t b) { return __vcmpltu2(a, b) != 0u; }
    // a distance (not only a pred) improved: what the delta pull propagates
    __device__ __forceinline__ static bool dist_less(uint32_t a, uint32_t b) {
        return __vcmpltu2(a | 0x000f000fu, b | 0x000f000fu) != 0u;
    }
    __device__ __forceinline__ static bool overflow(uint32_t d, uint32_t thr2) {
        return (__vcmpgeu2(d, thr2) & ~__vcmpeq2(d, INF)) != 0u;
    }
    __device__ __forceinline__ static uint32_t half(uint32_t x, int h) { return (x >> (16 * h)) & 0xffffu; }
    __device__ __forceinline__ static bool finite(uint32_t x1) { return x1 != INF1; }
    __device__ __forceinline__ static bool steep_tight(uint32_t du1, uint32_t w, uint32_t dv1) {
        return w != 0u && (du1 >> 4) + w == (dv1 >> 4);
    }
};

// --------------------------------------------------- per-lane row vectors --
template <int SPL>
struct Vec {
    uint32_t x[SPL];
};
template <int SPL>
__device__ __forceinline__ Vec<SPL> vload(const uint32_t *p) {
    Vec<SPL> r;
    if constexpr (SPL == 1) {
        r.x[0] = *p;
    } else if constexpr (SPL == 2) {
        const uint2 t = *reinterpret_cast<const uint2 *>(p);
        r.x[0] = t.x;
        r.x[1] = t.y;
    } else {
        const uint4 t = *reinterpret_cast<const uint4 *>(p);
        r.x[0] = t.x;
        r.x[1] = t.y;
        r.x[2] = t.z;
        r.x[3] = t.w;
    }
    return r;
}
template <int SPL>
__device__ __forceinline__ void vstore(uint32_t *p, const Vec<SPL> &v) {
    if constexpr (SPL == 1) {
        *p = v.x[0];
    } else if constexpr (SPL == 2) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(v.x[0], v.x[1]);
    } else {
        *reinterpret_cast<uint4 *>(p) = make_uint4(v.x[0], v.x[1], v.x[2], v.x[3]);
    }
}
template <class Op, int SPL>
__device__ __forceinline__ void vrelax(Vec<SPL> &d, const Vec<SPL> &x, uint32_t w) {
#pragma unroll
    for (int j = 0; j < SPL; ++j) d.x[j] = Op::relax(d.x[j], x.x[j], w);
}
template <class Op, int SPL>
__device__ __forceinline__ Vec<SPL> vmin(const Vec<SPL> &a, const Vec<SPL> &b) {
    Vec<SPL> r;
#pragma unroll
    for (int j = 0; j < SPL; ++j) r.x[j] = Op::min_word(a.x[j], b.x[j]);
    return r;
}
template <class Op, int SPL>
__device__ __forceinline__ bool vless(const Vec<SPL> &a, const Vec<SPL> &b) {
    bool r = false;
#pragma unroll
    for (int j = 0; j < SPL; ++j) r |= Op::any_less(a.x[j], b.x[j]);
    return r;
}

// ---------------------------------------------------- relaxing one word --
// Delta pull. In round r+1 a candidate only needs the in-arcs whose tail
// improved in round r: an in-neighbour that did not change since the
// candidate's previous relaxation was already folded in (if it changed
// after that read, it is in the changed set and comes back next round).
// The tails' change bits are tested lane-parallel (one bitmap probe per
// arc, ballot), and only the set arcs are gathered. Dense mode tests nothing.

// The change sets are round-stamped words (bits, round) in shared memory,
// double-buffered by round parity: a word written in round r is only read
// as "changed in round r" (stamp check), so stale words from earlier rounds
// never need clearing, and a word is written only when something changed.
struct ChgView {
    const uint2 *p;
    uint32_t r;   // the round whose changes are wanted
    __device__ __forceinline__ bool test(int u) const {
        const uint2 e = p[u >> 5];
        return e.y == r && ((e.x >> (u & 31)) & 1u);
    }
};

// Generic-degree pull of one vertex. Rl = this lane's first slot.
template <class Op, bool DELTA, int SPL>
__device__ __forceinline__ Vec<SPL> relax_vertex(const DevGraph &g, const uint32_t *__restrict__ Rl,
                                                 const ChgView pchg, int a0, int a1, int lane, Vec<SPL> d,
                                                 unsigned long long &relax) {
    constexpr int TSW = 32 * SPL;
    for (int base = a0; base < a1; base += 32) {
        const int cnt = min(32, a1 - base);
        int my_u = 0;
        uint32_t my_w = 0;
        bool take = false;
        if (lane < cnt) {
            my_u = g.in_src[base + lane];
            my_w = Op::prep_w(g.in_w[base + lane], base - a0 + lane);
            take = !DELTA || pchg.test(my_u);
        }
        uint32_t m = __ballot_sync(FULL, take);
        relax += (unsigned long long)__popc(m);
        while (m) {
            const int k0 = __ffs(m) - 1;
            m &= m - 1;
            const bool two = m != 0;
            const int k1 = two ? __ffs(m) - 1 : k0;
            if (two) m &= m - 1;
            const int u0 = __shfl_sync(FULL, my_u, k0), u1 = __shfl_sync(FULL, my_u, k1);
            const uint32_t w0 = __shfl_sync(FULL, my_w, k0), w1 = __shfl_sync(FULL, my_w, k1);
            const Vec<SPL> x0 = vload<SPL>(Rl + (size_t)u0 * TSW);
            Vec<SPL> x1 = x0;
            if (two) x1 = vload<SPL>(Rl + (size_t)u1 * TSW);
            vrelax<Op, SPL>(d, x0, w0);
            if (two) vrelax<Op, SPL>(d, x1, w1);
        }
    }
    return d;
}

// Relaxes the candidate vertices (bits of m) of word w for every slot, in
// three steps that keep the control work lane-parallel:
//  A. lane = candidate vertex: walk its in-arcs, test each tail's change bit
//     (delta pull) and append the changed arcs (u, w) to the lane's slots of
//     the warp's task queue in shared memory (<= QCAP per vertex, else the
//     vertex takes the generic path);
//  B. lane = source slots: for the candidate vertices two at a time, load
//     their own rows and gather the queued tails' rows (up to four gathers
//     in flight), min-plus relax, store improved rows, vote;
//  C. lane = vertex again: every improved vertex marks its out-neighbours in
//     the next round's candidate bitmap (shared-memory atomicOr); the lane
//     that turns a word non-zero appends it to the next round's word list.
// Returns the word's change mask.
// Task-queue capacity per vertex: per-warp queues of 32 x QC packed (u, w)
// pairs after the bitmaps in dynamic shared memory.
#ifndef WR_QCAP
#define WR_QCAP 12   // C5's in-degree is <= 10; more changed in-arcs take relax_vertex
#endif
constexpr int QCAP = WR_QCAP;
#ifndef WR_AQ
#define WR_AQ 8   // in-arcs loaded per batch in step A
#endif
#ifndef WR_FUSED_PA
#define WR_FUSED_PA 2
#endif
constexpr int FPA = WR_FUSED_PA;   // in-arcs per vertex per step in the fused pred jobs (1: 65.0 ms, 2: 64.0, 3: 65.6)

// Near-far state of one CTA (NF kernels only): the deferred bitmap and the
// inlist bitmaps live in shared memory, keys and word lists in global.
struct NfState {
    uint32_t *pend;      // [NW] deferred vertices
    uint32_t *inl;       // [2][NWB] words already in list 0 / 1
    uint32_t *keys;      // [V] min deferred key (fp32 bits)
    int *plist;          // [2][NW] words with deferred vertices
    int *plen;           // [2] (shared)
    int cur;             // list being filled this round
    float T;             // threshold
};

__device__ __forceinline__ void nf_append(NfState &nf, int which, int w, int NW) {
    const uint32_t b = 1u << (w & 31);
    if (!(atomicOr(&nf.inl[which * ((NW + 31) >> 5) + (w >> 5)], b) & b))
        nf.plist[which * NW + atomicAdd(&nf.plen[which], 1)] = w;
}

template <class Op, bool DELTA, int SPL, int QC, int VB, int TPS, bool LIST, bool NF = false>
__device__ __forceinline__ uint32_t relax_word(const DevGraph &g, uint32_t *__restrict__ R, int w, uint32_t m,
                                               int lane, unsigned long long &relax, const ChgView pchg,
                                               uint32_t *nxt, uint16_t *nlist, int *nlen, int2 *q,
                                               uint32_t *touched, bool &ovf, uint32_t thr2,
                                               NfState *nfp = nullptr) {
    constexpr int TSW = 32 * SPL;
    const int v = (w << 5) + lane;
    const bool act = (m >> lane) & 1u;
    int a0 = 0, a1 = 0, o0 = 0, o1 = 0;
    if (act) {   // out-arc range loaded now: step C then needs one dependent load less
        a0 = g.in_ptr[v];
        a1 = g.in_ptr[v + 1];
        if (DELTA) {
            o0 = g.out_ptr[v];
            o1 = g.out_ptr[v + 1];
        }
    }
    // ---- A: queue this lane's changed in-arcs; the packed (u, w) arcs are
    // loaded AQ at a time (independent loads in flight, no branch between
    // them) before their tails' change bits are tested
    constexpr int AQ = WR_AQ;
    int c = 0;
    for (int k0 = a0; k0 < a1; k0 += AQ) {
        int2 arc[AQ];
#pragma unroll
        for (int j = 0; j < AQ; ++j) arc[j] = (k0 + j < a1) ? g.in_arc[k0 + j] : make_int2(-1, 0);
#pragma unroll
        for (int j = 0; j < AQ; ++j) {
            const bool take = arc[j].x >= 0 && (!DELTA || pchg.test(arc[j].x));
            // queued: the tail row's byte offset (u * TSW * 4 < 2^31 for V within the frontier limit)
            if (take && c < QC) q[lane * QC + c] = make_int2(arc[j].x * (TSW * 4), (int)Op::prep_w((uint32_t)arc[j].y, k0 + j - a0));
            c += take ? 1 : 0;
        }
    }
    relax += (unsigned long long)__reduce_add_sync(FULL, (unsigned)c);
    __syncwarp();
    uint32_t todo = __ballot_sync(FULL, c > 0);
    // rows are written lazily: a vertex never improved so far holds no row
    // yet and reads as INF (its first improvement writes the whole row)
    const uint32_t tw = DELTA ? touched[w] : FULL;
    Vec<SPL> infv;
#pragma unroll
    for (int j = 0; j < SPL; ++j) infv.x[j] = Op::INF;
    const uint32_t slow = __ballot_sync(FULL, c > QC);
    uint32_t *Rl = R + lane * SPL;
    uint32_t chg = 0, wrote = 0;
    unsigned long long dummy = 0;
    // ---- B: relax the queued vertices, VB per step, TPS tasks each per
    // step (VB*TPS row gathers in flight)
    while (todo) {
        int iv[VB];
        bool ok[VB];
#pragma unroll
        for (int k = 0; k < VB; ++k) {
            ok[k] = todo != 0;
            iv[k] = ok[k] ? __ffs(todo) - 1 : 0;
            if (ok[k]) todo &= todo - 1;
        }
        Vec<SPL> e[VB], d[VB];
        int cc[VB];
        bool anyslow = false;
#pragma unroll
        for (int k = 0; k < VB; ++k) {
            // the own row is only needed at the end: d starts at INF so the
            // row loads overlap the tails' gathers instead of preceding them
            e[k] = infv;
            if (ok[k] && ((tw >> iv[k]) & 1u)) e[k] = vload<SPL>(Rl + (size_t)((w << 5) + iv[k]) * TSW);
            d[k] = infv;
            cc[k] = __shfl_sync(FULL, c, iv[k]);
            if (!ok[k]) cc[k] = 0;
            anyslow |= ok[k] && ((slow >> iv[k]) & 1u);
        }
        if (!anyslow) {
            int tmax = 0;
#pragma unroll
            for (int k = 0; k < VB; ++k) tmax = max(tmax, cc[k]);
            const char *Rb = reinterpret_cast<const char *>(Rl);
            for (int t = 0; t < tmax; t += TPS) {
                int2 tk[VB][TPS];
                Vec<SPL> x[VB][TPS];
                // queue entries are read unconditionally (stale entries past
                // cc are valid shared memory, never used): no zero-fill, and
                // two entries per 16-B load
#pragma unroll
                for (int k = 0; k < VB; ++k) {
                    if constexpr (TPS == 2 && QC % 2 == 0) {
                        const int4 two = *reinterpret_cast<const int4 *>(q + iv[k] * QC + min(t, QC - 2));
                        tk[k][0] = make_int2(two.x, two.y);
                        tk[k][1] = make_int2(two.z, two.w);
                    } else {
#pragma unroll
                        for (int j = 0; j < TPS; ++j) tk[k][j] = q[iv[k] * QC + min(t + j, QC - 1)];
                    }
                }
#pragma unroll
                for (int k = 0; k < VB; ++k)
#pragma unroll
                    for (int j = 0; j < TPS; ++j)
                        if (t + j < cc[k])
                            x[k][j] = vload<SPL>(reinterpret_cast<const uint32_t *>(Rb + (uint32_t)tk[k][j].x));
#pragma unroll
                for (int k = 0; k < VB; ++k)
#pragma unroll
                    for (int j = 0; j < TPS; ++j)
                        if (t + j < cc[k]) vrelax<Op, SPL>(d[k], x[k][j], (uint32_t)tk[k][j].y);
            }
        } else {
#pragma unroll
            for (int k = 0; k < VB; ++k) {
                if (!ok[k]) continue;
                if ((slow >> iv[k]) & 1u) {
                    d[k] = relax_vertex<Op, DELTA, SPL>(g, Rl, pchg, __shfl_sync(FULL, a0, iv[k]),
                                                        __shfl_sync(FULL, a1, iv[k]), lane, d[k], dummy);
                } else {
                    for (int t = 0; t < cc[k]; ++t) {
                        const int2 tq = q[iv[k] * QC + t];
                        vrelax<Op, SPL>(d[k], vload<SPL>(reinterpret_cast<const uint32_t *>(
                                                  reinterpret_cast<const char *>(Rl) + (uint32_t)tq.x)),
                                        (uint32_t)tq.y);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < VB; ++k) {
            // nv = min(new, own row): the row improved iff some word of nv
            // differs from the own row (one min + one xor per word instead
            // of emulated per-half compares); keyed rows propagate only when
            // a distance (not just a pred index) improved
            const Vec<SPL> nv = vmin<Op, SPL>(d[k], e[k]);
            uint32_t diff = 0, ddiff = 0;
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                const uint32_t x = nv.x[j] ^ e[k].x[j];
                diff |= x;
                if constexpr (Op::KEYED) ddiff |= x & 0xfff0fff0u;
            }
            // first write of a row covers every slot (untouched slots stay INF)
            const bool f = ok[k] && !((tw >> iv[k]) & 1u);
            const bool lt = ok[k] && diff != 0u;                   // the row improved (store it)
            bool ch = Op::KEYED ? ok[k] && ddiff != 0u : lt;        // a distance improved (propagate)
            if (__any_sync(FULL, lt)) wrote |= 1u << iv[k];
            if constexpr (NF) {
                // near-far: defer the propagation while every improved slot
                // is beyond T (the row is stored either way)
                if (__any_sync(FULL, ch)) {
                    uint32_t km = 0xffffffffu;   // fp32 >= 0: bit order = value order
#pragma unroll
                    for (int j = 0; j < SPL; ++j)
                        if (nv.x[j] != e[k].x[j]) km = min(km, nv.x[j]);
                    km = __reduce_min_sync(FULL, km);
                    NfState &nf = *nfp;
                    const uint32_t bit = 1u << iv[k];
                    const int vv = (w << 5) + iv[k];
                    if (__uint_as_float(km) > nf.T) {
                        ch = false;
                        if (lane == 0) {   // this warp owns word w this round
                            const uint32_t old = nf.pend[w];
                            nf.keys[vv] = (old & bit) ? min(nf.keys[vv], km) : km;
                            nf.pend[w] = old | bit;
                            if (!old) nf_append(nf, nf.cur, w, (g.V + 31) >> 5);
                        }
                    } else if (lane == 0 && (nf.pend[w] & bit)) {
                        nf.pend[w] &= ~bit;   // propagated now, with everything deferred before
                    }
                }
            }
            if (lt || f) {
                vstore<SPL>(Rl + (size_t)((w << 5) + iv[k]) * TSW, nv);
                // keyed rows are range-checked by the pred jobs instead (every key is decoded there)
                if constexpr (Op::PACK > 1 && !Op::KEYED) {
#pragma unroll
                    for (int j = 0; j < SPL; ++j) ovf |= Op::overflow(nv.x[j], thr2);
                }
            }
            if (__any_sync(FULL, ch)) chg |= 1u << iv[k];
        }
    }
    if (DELTA && lane == 0 && (wrote & ~tw)) touched[w] = tw | wrote;   // this warp owns word w
    // ---- C: improved vertices mark their out-neighbours, lane-parallel
    if (DELTA && ((chg >> lane) & 1u)) {
        for (int e = o0; e < o1; ++e) {
            const int x = g.out_dst[e];
            if (LIST) {
                if (atomicOr(&nxt[x >> 5], 1u << (x & 31)) == 0u) nlist[atomicAdd(nlen, 1)] = (uint16_t)(x >> 5);
            } else {
                atomicOr(&nxt[x >> 5], 1u << (x & 31));
            }
        }
    }
    __syncwarp();   // the queue is reused by the warp's next word
    return chg;
}

// ------------------------------------------------------ the sweep kernel --
// One CTA per tile at a time. Shared memory (frontier variant):
//   cur, nxt   V-bit candidate bitmaps (relaxed this round / out-neighbours
//              of this round's improvements), swapped each round;
//   touched    vertices whose row has been written (lazy rows);
//   chg[2]     round-stamped change words (ChgView), by round parity;
//   list[2]    the non-zero words of cur / nxt (16-bit word indices), so a round visits only its
//              candidate words, handed out to warps dynamically (one shared
//              counter per round) - no scan over all V/32 words and no
//              static word-to-warp split that leaves warps idle at the
//              round barrier;
//   queues     per-warp task queues (relax_word).
// Dense variant: every vertex is a candidate every round, all arcs pulled
// (the paper's edge-parallel class of work), words split statically.
struct FrontierSmem {
    size_t cur, nxt, touched, chg, list, queue, words;
};
__host__ __device__ constexpr FrontierSmem frontier_smem(int NW, int nwarps, int QC) {
    // offsets in 32-bit words; uint2 / int2 regions 8-B aligned
    // (the task queues start 16-B aligned: step B reads two entries per int4)
    return FrontierSmem{0,
                        (size_t)NW,
                        (size_t)2 * NW,
                        ((size_t)3 * NW + 1) & ~(size_t)1,
                        (((size_t)3 * NW + 1) & ~(size_t)1) + (size_t)4 * NW,
                        ((((size_t)3 * NW + 1) & ~(size_t)1) + (size_t)5 * NW + 3) & ~(size_t)3,
                        (((((size_t)3 * NW + 1) & ~(size_t)1) + (size_t)5 * NW + 3) & ~(size_t)3) +
                            (size_t)nwarps * 32 * QC * 2};
}

struct PredShape {
    static constexpr int PV = 8;     // vertices per warp job (full 32-B output sectors)
};
template <class Op, int SPL, int PA>
__device__ __forceinline__ void pred_job(const DevGraph &g, const int *__restrict__ tile_src,
                                         const uint32_t *__restrict__ rows, const int *__restrict__ slot_row,
                                         int64_t out_row0, int32_t *__restrict__ pred_out, int *flat_tiles, int tile,
                                         int c0, int32_t *spw, int lane);

// keyed staging rows: slot s at s + s / 32 (a skew that makes both the
// per-lane writes of 8 consecutive slots and the per-slot reads conflict-free)
template <int TS_>
struct SkewStage {
    static constexpr int TS = TS_;
    static constexpr int RS = TS + TS / 32 + 1;
    __device__ static int at(int s) { return s + (s >> 5); }
};
// keyed pred jobs stage in-arc indices, not vertex ids: per vertex one word
// per lane holding its 2 SPL slots' 4-bit indices, plus the vertex's in-arc
// tails (<= 16) - 48 words per vertex instead of 265, which keeps the fused
// kernel's shared memory (and so its L1 carveout) at the frontier's size
struct KeyedStage {
    static constexpr int WORDS = 32 + 16;   // per vertex: packed indices, tails
};
template <int SPL>
__device__ __forceinline__ void pred_job_keyed(const DevGraph &g, const int *__restrict__ tile_src,
                                               const uint32_t *__restrict__ rows, const int *__restrict__ slot_row,
                                               int64_t out_row0, int32_t *__restrict__ pred_out, int tile, int c0,
                                               int32_t *spw, int lane, uint32_t thr, int *overflow,
                                               int (&srow)[2 * SPL], int &srow_tile);


template <class Op, bool DENSE, int NT, int MINB, int SPL, int QC, int VB, int TPS, bool LIST, bool NF = false>
__global__ void __launch_bounds__(NT, MINB) bf_frontier_kernel(DevGraph g, const int *__restrict__ tile_src,
                                                               int ntiles, uint32_t *__restrict__ rows,
                                                               int *tile_counter, int max_rounds,
                                                               BfTileStats *stats, uint32_t thr2,
                                                               const int *__restrict__ tile_order, PredFuse fuse,
                                                               const int *__restrict__ slot_row, NearFar nfa) {
    constexpr int TSW = 32 * SPL;              // 32-bit words per row
    constexpr int TS = TSW * Op::PACK;         // sources per tile
    constexpr int NWARPS = NT / 32;
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ int s_tile;
    __shared__ int s_len[3], s_head[3];
    __shared__ int s_plen[2], s_phead;
    __shared__ uint32_t s_kmin;
    const int V = g.V;
    const int NW = (V + 31) >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t last_mask = (V & 31) ? ((1u << (V & 31)) - 1u) : 0xffffffffu;
    const FrontierSmem L = frontier_smem(NW, NWARPS, QC);
    uint32_t *const touched = smem + L.touched;
    uint2 *const chg = reinterpret_cast<uint2 *>(smem + L.chg);
    uint16_t *const list = reinterpret_cast<uint16_t *>(smem + L.list);   // NW < 2^16 (launch_shape)
    int2 *const q = reinterpret_cast<int2 *>(smem + L.queue) + warp * (32 * QC);
    const int NWB = (NW + 31) >> 5;
    NfState nf{};
    if constexpr (NF) {   // after the queues: pend[NW], inl[2][NWB]
        nf.pend = smem + L.words;
        nf.inl = nf.pend + NW;
        nf.keys = nfa.keys + (size_t)blockIdx.x * V;
        nf.plist = nfa.plist + (size_t)blockIdx.x * 2 * NW;
        nf.plen = s_plen;
    }

    for (;;) {
        if (threadIdx.x == 0) {
            const int k = atomicAdd(tile_counter, 1);
            s_tile = (k < ntiles && tile_order) ? tile_order[k] : k;
        }
        __syncthreads();
        const int tile = s_tile;
        if (tile >= ntiles) break;
        long long t_start = 0;
        if (fuse.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        uint32_t *R = rows + (size_t)tile * V * TSW;
        uint32_t *cur = smem + L.cur, *nxt = smem + L.nxt;

        // init: bitmaps and stamps zero (round 0 = the seeds); rows INF
        // (dense) or written lazily (frontier: a row is written whole on its
        // vertex's first improvement, and the rows of vertices never reached
        // are filled with INF at the end)
        const uint4 inf4 = make_uint4(Op::INF, Op::INF, Op::INF, Op::INF);
        if (DENSE) {
            uint4 *R4 = reinterpret_cast<uint4 *>(R);
            const size_t n4 = (size_t)V * (TSW / 4);
            for (size_t i = threadIdx.x; i < n4; i += NT) R4[i] = inf4;
        }
        for (size_t i = threadIdx.x; i < L.list; i += NT) smem[i] = 0u;
        if (threadIdx.x < 3) s_len[threadIdx.x] = s_head[threadIdx.x] = 0;
        if constexpr (NF) {
            for (int i = threadIdx.x; i < NW + 2 * NWB; i += NT) nf.pend[i] = 0u;
            if (threadIdx.x < 2) s_plen[threadIdx.x] = 0;
            nf.cur = 0;
            nf.T = nfa.delta;
        }
        __syncthreads();
        if (warp == 0) {   // seed: d[s][slot] = 0; the sources "changed" in round 0
            if (!DENSE) {  // the seed vertices' rows: INF everywhere first
                for (int k = 0; k < TS; ++k) {
                    const int s = tile_src[tile * TS + k];
                    if (s >= 0) {
                        uint32_t *row = R + (size_t)s * TSW;
                        for (int c = lane; c < TSW / 4; c += 32) reinterpret_cast<uint4 *>(row)[c] = inf4;
                    }
                }
                __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < SPL * Op::PACK; ++j) {
                const int slot = lane * SPL * Op::PACK + j;
                const int s = tile_src[tile * TS + slot];
                if (s >= 0) {
                    if constexpr (Op::PACK == 1) R[(size_t)s * TSW + slot] = Op::ZERO;
                    else reinterpret_cast<uint16_t *>(R)[(size_t)s * TS + slot] = Op::SEED16;
                    atomicOr(&chg[s >> 5].x, 1u << (s & 31));   // stamp 0 = round 0
                    atomicOr(&touched[s >> 5], 1u << (s & 31));
                    for (int e = g.out_ptr[s]; e < g.out_ptr[s + 1]; ++e) {
                        const int x = g.out_dst[e];
                        if (atomicOr(&cur[x >> 5], 1u << (x & 31)) == 0u) list[NW + atomicAdd(&s_len[1], 1)] = (uint16_t)(x >> 5);
                    }
                }
            }
        }
        __syncthreads();

        int rounds = 0;
        unsigned long long relax = 0, visits = 0;
        bool more = true, ovf = false;
        for (int r = 1; more; ++r) {
            int any = 0;
            if (DENSE) {
                for (int w = threadIdx.x; w < NW; w += NT) cur[w] = (w == NW - 1) ? last_mask : 0xffffffffu;
                __syncthreads();
                for (int w = warp; w < NW; w += NWARPS) {
                    const uint32_t m = cur[w];
                    const uint32_t c = relax_word<Op, false, SPL, QC, VB, TPS, false>(
                        g, R, w, m, lane, relax, ChgView{chg, 0u}, nxt, list, &s_len[0], q, touched, ovf, thr2);
                    visits += (unsigned long long)__popc(m);
                    any |= c != 0;
                }
            } else if (!LIST) {
                // ---- static split: warp k scans words k, k + NWARPS, ...
                const ChgView pc{chg + ((r - 1) & 1) * NW, (uint32_t)(r - 1)};
                uint2 *cc = chg + (r & 1) * NW;
                for (int w = warp; w < NW; w += NWARPS) {
                    const uint32_t m = cur[w];
                    if (!m) continue;
                    __syncwarp();
                    if (lane == 0) cur[w] = 0u;
                    const uint32_t c = relax_word<Op, true, SPL, QC, VB, TPS, false, NF>(
                        g, R, w, m, lane, relax, pc, nxt, nullptr, nullptr, q, touched, ovf, thr2, &nf);
                    if (lane == 0 && c) cc[w] = make_uint2(c, (uint32_t)r);
                    visits += (unsigned long long)__popc(m);
                    any |= c != 0;
                }
            } else {
                // ---- relax the candidate words of list r&1, claimed one at a
                // time; improvements append to list (r+1)&1
                const uint16_t *lc = list + (r & 1) * NW;
                uint16_t *ln = list + ((r + 1) & 1) * NW;
                const int len = s_len[r % 3];
                int *const nlen = &s_len[(r + 1) % 3];
                if (threadIdx.x == 0) s_len[(r + 2) % 3] = s_head[(r + 2) % 3] = 0;   // used in round r-1
                const ChgView pc{chg + ((r - 1) & 1) * NW, (uint32_t)(r - 1)};
                uint2 *cc = chg + (r & 1) * NW;
                for (;;) {
                    int i = 0;
                    if (lane == 0) i = atomicAdd(&s_head[r % 3], 1);
                    i = __shfl_sync(FULL, i, 0);
                    if (i >= len) break;
                    const int w = lc[i];
                    const uint32_t m = cur[w];
                    __syncwarp();
                    if (lane == 0) cur[w] = 0u;
                    const uint32_t c = relax_word<Op, true, SPL, QC, VB, TPS, true, NF>(
                        g, R, w, m, lane, relax, pc, nxt, ln, nlen, q, touched, ovf, thr2, &nf);
                    if (lane == 0 && c) cc[w] = make_uint2(c, (uint32_t)r);
                    visits += (unsigned long long)__popc(m);
                    any |= c != 0;
                }
            }
            bool nf_released = false;
            if constexpr (NF) {
                uint2 *cc = chg + (r & 1) * NW;
                uint16_t *ln = LIST ? list + ((r + 1) & 1) * NW : nullptr;
                int *const nlen = LIST ? &s_len[(r + 1) % 3] : nullptr;
                // near-far release: deferred vertices whose key is <= T
                    // now propagate as if they had changed in round r (change
                    // bits stamped r, out-neighbours into round r+1's list);
                    // when nothing is near, T jumps to the nearest deferred key
                    const bool near0 = __syncthreads_or(any) != 0;   // this round propagated something
                    bool released = false;
                    for (;;) {
                        const int src = nf.cur, dst = nf.cur ^ 1;
                        if (threadIdx.x == 0) { s_plen[dst] = 0; s_phead = 0; s_kmin = 0xffffffffu; }
                        for (int i = threadIdx.x; i < NWB; i += NT) nf.inl[dst * NWB + i] = 0u;
                        __syncthreads();
                        const int plen = s_plen[src];
                        for (;;) {
                            int i = 0;
                            if (lane == 0) i = atomicAdd(&s_phead, 1);
                            i = __shfl_sync(FULL, i, 0);
                            if (i >= plen) break;
                            const int w = nf.plist[src * NW + i];
                            const uint32_t bits = nf.pend[w];
                            const int v = (w << 5) + lane;
                            uint32_t key = 0xffffffffu;
                            if ((bits >> lane) & 1u) key = nf.keys[v];
                            const bool rel = ((bits >> lane) & 1u) && __uint_as_float(key) <= nf.T;
                            const uint32_t relm = __ballot_sync(FULL, rel), keep = bits & ~relm;
                            if (rel) {   // mark the out-neighbours for round r+1
                                for (int e2 = g.out_ptr[v]; e2 < g.out_ptr[v + 1]; ++e2) {
                                    const int x = g.out_dst[e2];
                                    if (atomicOr(&nxt[x >> 5], 1u << (x & 31)) == 0u && LIST) ln[atomicAdd(nlen, 1)] = (uint16_t)(x >> 5);
                                }
                            }
                            const uint32_t kk = __reduce_min_sync(FULL, ((keep >> lane) & 1u) ? key : 0xffffffffu);
                            if (lane == 0) {
                                if (relm) {
                                    const uint2 e0 = cc[w];
                                    cc[w] = e0.y == (uint32_t)r ? make_uint2(e0.x | relm, (uint32_t)r)
                                                                : make_uint2(relm, (uint32_t)r);
                                }
                                nf.pend[w] = keep;
                                if (keep) {
                                    nf_append(nf, dst, w, NW);
                                    atomicMin(&s_kmin, kk);
                                }
                            }
                            released |= relm != 0u;
                        }
                        __syncthreads();
                        nf.cur = dst;
                        // T advances by delta per round; with nothing near it
                        // jumps to the nearest deferred key and releases again
                        released = __syncthreads_or(released) != 0;
                        const bool near = near0 || released, pending = s_plen[dst] > 0;
                        if (near || !pending) {
                            nf.T += nfa.delta;
                            nf_released = released;
                            break;
                        }
                        nf.T = fmaxf(nf.T + nfa.delta, __uint_as_float(s_kmin));
                    }
                }
            ++rounds;
            any |= nf_released;
            more = __syncthreads_or(any) != 0;
            uint32_t *t = cur;
            cur = nxt;
            nxt = t;
            // max_rounds relaxation rounds (P724 §4.7: V-1), then one more
            // round as the check pass (the oracle's extra pass): a change in
            // round max_rounds + 1 means a negative cycle (or, for a caller's
            // smaller max_rounds, no convergence)
            if (more && rounds > max_rounds) {
                if (threadIdx.x == 0) atomicMax(&stats->negcycle_tile, tile);
                more = false;
            }
        }
        if (!DENSE) {   // vertices never reached: their rows read INF
            for (int w = warp; w < NW; w += NWARPS) {
                uint32_t um = ~touched[w] & (w == NW - 1 ? last_mask : FULL);
                while (um) {
                    const int b = __ffs(um) - 1;
                    um &= um - 1;
                    uint4 *row = reinterpret_cast<uint4 *>(R + (size_t)((w << 5) + b) * TSW);
                    for (int c = lane; c < TSW / 4; c += 32) row[c] = inf4;
                }
            }
        }
        if (Op::PACK > 1 && __syncthreads_or(ovf) && threadIdx.x == 0) atomicOr(&stats->overflow, 1);
        // per-tile statistics (one lane per warp contributes its arc count)
        if (lane == 0 && relax) atomicAdd(&stats->relax, relax * TS);
        if (lane == 0 && visits) atomicAdd(&stats->visits, visits);
        if (threadIdx.x == 0) atomicMax(&stats->rounds_max, rounds);
        if (fuse.trace && threadIdx.x == 0) {   // diagnostics (WR_TILE_TRACE)
            long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            long long *e = fuse.trace + 4 * (size_t)tile;
            e[0] = t_start;
            e[1] = t_end;
            e[2] = rounds;
            e[3] = smid;
        }
        if (fuse.pred_out) {   // publish the finished tile: rows visible GPU-wide, then its list entry
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                const int k = atomicAdd(&fuse.counters[0], 1);
                asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(fuse.done_list + k), "r"(tile) : "memory");
            }
        }
        __syncthreads();
    }
    if (fuse.trace && threadIdx.x == 0) {   // diagnostics: this CTA's sweep end / pred-jobs end
        long long t_now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
        fuse.trace[4 * (size_t)ntiles + 2 * blockIdx.x] = t_now;
    }
    if (fuse.pred_out && !DENSE) {
        // no tile left to claim: take pred jobs (tile in completion order k,
        // 8-vertex chunk) - a job waits only for a tile that a running CTA
        // is still relaxing; the shared memory is free for the staging rows
        constexpr int PV = PredShape::PV;
        const int chunks = (V + PV - 1) / PV;
        const long long njobs = (long long)ntiles * chunks;
        int srow_cache[2 * SPL], srow_tile = -1;   // keyed jobs: output rows of the current tile's slots
#ifndef WR_PRED_JB
#define WR_PRED_JB 1   // jobs per claim; C5: 1 -> 57.7 ms/step, 4 -> 63.3 (consecutive chunks on one warp serialise)
#endif
        constexpr int JB = WR_PRED_JB;
        long long jnext = 0, jend = 0;
        int kcur = -1, t = -1;
        for (;;) {
            if (jnext >= jend) {
                long long j0 = 0;
                if (lane == 0)
                    j0 = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(fuse.counters + 2),
                                              (unsigned long long)JB);
                jnext = __shfl_sync(FULL, j0, 0);
                jend = jnext + JB;
            }
            const long long j = jnext++;
            if (j >= njobs) break;
            const int k = (int)(j / chunks);
            if (k != kcur) {   // wait until tile k (in completion order) is done
                if (lane == 0) {
                    // poll relaxed (an acquire load invalidates the SM's L1 on
                    // every try), then one acquire once the tile is published
                    for (;;) {
                        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(t) : "l"(fuse.done_list + k) : "memory");
                        if (t >= 0) break;
                        __nanosleep(256);
                    }
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(t) : "l"(fuse.done_list + k) : "memory");
                }
                t = __shfl_sync(FULL, t, 0);
                kcur = k;
            }
            if constexpr (Op::KEYED)
                pred_job_keyed<SPL>(g, tile_src, rows, slot_row, fuse.out_row0, fuse.pred_out, t,
                                    (int)(j % chunks) * PV,
                                    reinterpret_cast<int32_t *>(smem) + warp * PV * KeyedStage::WORDS, lane,
                                    thr2 & 0xffffu, &stats->overflow, srow_cache, srow_tile);
            else
                pred_job<Op, SPL, FPA>(g, tile_src, rows, slot_row, fuse.out_row0, fuse.pred_out, fuse.flat_tiles, t,
                                       (int)(j % chunks) * PV,
                                       reinterpret_cast<int32_t *>(smem) + warp * PV * SkewStage<TS>::RS, lane);
        }
    }
    if (fuse.trace && threadIdx.x == 0) {
        long long t_now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
        fuse.trace[4 * (size_t)ntiles + 2 * blockIdx.x + 1] = t_now;
    }
}

static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

// Launch shapes (threads per CTA, min CTAs per SM) compiled for the sweep;
// WR_BF_CONFIG selects one (tuning knob; default measured best).
template <class Op, bool DENSE, int NT, int MINB, int SPL, int QC = QCAP, bool LIST = false, int VB = 2, int TPS = 2,
          bool NF = false>
static bool launch_shape(const wr_graph *g, const BfRun &run, BfTileStats *d_stats, cudaStream_t st) {
    auto kern = bf_frontier_kernel<Op, DENSE, NT, MINB, SPL, QC, VB, TPS, LIST && !DENSE, NF>;
    const int NW = (g->V + 31) / 32;
    if (NW > 65535) return false;   // 16-bit word lists
    size_t smem = frontier_smem(NW, NT / 32, QC).words * sizeof(uint32_t);
    if (NF) smem += (size_t)(NW + 2 * ((NW + 31) / 32)) * sizeof(uint32_t);   // deferred bitmap + inlist bitmaps
    if (run.fuse.pred_out)   // the fused pred jobs' staging rows reuse it
        smem = std::max(smem, (size_t)(NT / 32) * PredShape::PV *
                                  (Op::KEYED ? KeyedStage::WORDS : SkewStage<32 * SPL * Op::PACK>::RS) *
                                  sizeof(int32_t));
    smem += (size_t)env_int("WR_SMEM_PAD", 0);   // experiment knob: less L1 (carveout study)
    int max_optin = 0;
    WR_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
    if (smem > (size_t)max_optin) return false;
    WR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, nsm = 0;
    WR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    WR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    per_sm = std::max(per_sm, 1);
    int grid = (int)std::min<int64_t>(run.ntiles, (int64_t)per_sm * nsm);
    if (const int cap = env_int("WR_BF_GRID", 0)) grid = std::max(1, std::min(grid, cap));   // experiment knob
    DBuf<int> counter(1);
    WR_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(int), st));
    NearFar nfa;
    DBuf<uint32_t> nf_keys;
    DBuf<int> nf_plist;
    if (NF) {   // per persistent CTA: keys[V], two word lists
        nf_keys.alloc((size_t)grid * g->V);
        nf_plist.alloc((size_t)grid * 2 * NW);
        nfa.keys = nf_keys.p;
        nfa.plist = nf_plist.p;
        nfa.delta = run.nf_delta;
    }
    kern<<<grid, NT, smem, st>>>(g->view(), run.tile_src, run.ntiles, run.rows, counter.p, run.max_rounds, d_stats,
                                 run.ovf_thr * 0x10001u, run.tile_order, run.fuse, run.slot_row, nfa);
    count_launch();
    WR_LAUNCH_CHECK();
    return true;   // the counter goes back to the stream-ordered pool: no sync needed
}


template <class Op, bool DENSE, int SPL>
static void launch_dispatch(const wr_graph *g, const BfRun &run, BfTileStats *d_stats, cudaStream_t st) {
    // (640 threads with 3x2 / 2x3 gathers per step, 512 threads with 2x4 /
    // 4x2: 61-78 ms, spills; 2x2 at 640: 42.7 ms)
    // launch shapes measured on config 5; 1 CTA per SM keeps
    // the tiles in flight (L2 working set) at one per SM. int32 sweep:
    // 768 threads + word lists (14) 77.6 ms, 768 static (8) 80.6, 640 lists
    // (11) 84.4, 640 static (9) 94.4, 896 static (10) 104; fp32: 768 static
    // 232 ms, 640 static 240, 768 lists 254 (the list order lets more
    // suboptimal values propagate: 4.4 vs 3.6 x S*E relaxations).
    // (the other shapes measured there - 384 x 2, 896, 704/768 with lists -
    // were dropped from the build; WR_BF_CONFIG picks 8 or 11. Round 2,
    // after the leaner task loop, keyed C5: 640 x (2 vertices x 2 tasks)
    // 62.1 ms/step; 640 x 3x2 65.7 (spills), 512 x 3x2 63.9, 512 x 4x2 70.3,
    // 768 x 2x2 63.4 - more gathers per warp do not pay at 96 registers)
    static const int cfg = env_int("WR_BF_CONFIG", std::is_same<Op, OpF32>::value ? 8 : 11);
    bool ok = false;
    if constexpr (std::is_same<Op, OpF32>::value && !DENSE) {   // near-far deferral (NEXT-3)
        if (run.nf_delta > 0.f) {
            static const int nfcfg = env_int("WR_NF_CONFIG", 8);
            if (nfcfg == 8 && launch_shape<Op, DENSE, 768, 1, SPL, QCAP, false, 2, 2, true>(g, run, d_stats, st)) return;
            if (launch_shape<Op, DENSE, 640, 1, SPL, QCAP, true, 2, 2, true>(g, run, d_stats, st)) return;
        }
    }
    switch (cfg) {
        case 8: ok = launch_shape<Op, DENSE, 768, 1, SPL>(g, run, d_stats, st); break;
        case 11: ok = launch_shape<Op, DENSE, 640, 1, SPL, QCAP, true>(g, run, d_stats, st); break;
        default: break;
    }
    if (!ok && !launch_shape<Op, DENSE, 640, 1, SPL>(g, run, d_stats, st) &&
        !launch_shape<Op, DENSE, 256, 1, SPL, 4>(g, run, d_stats, st))
        WR_THROW(WR_ETOOLARGE, "bf: V too large for the shared-memory frontier bitmaps");
}

template <class Op>
static void launch_sweep(const wr_graph *g, const BfRun &run, BfTileStats *d_stats, cudaStream_t st) {
    // packed rows serve the routing path only, which never asks for dense
    const bool dense = Op::PACK == 1 && run.variant == WR_BF_DENSE;
    switch (run.spl) {
        case 4:
            if constexpr (Op::PACK == 1) if (dense) { launch_dispatch<Op, true, 4>(g, run, d_stats, st); break; }
            launch_dispatch<Op, false, 4>(g, run, d_stats, st);
            break;
        case 2:
            if constexpr (Op::PACK == 1) if (dense) { launch_dispatch<Op, true, 2>(g, run, d_stats, st); break; }
            launch_dispatch<Op, false, 2>(g, run, d_stats, st);
            break;
        default:
            if constexpr (Op::PACK == 1) if (dense) { launch_dispatch<Op, true, 1>(g, run, d_stats, st); break; }
            launch_dispatch<Op, false, 1>(g, run, d_stats, st);
            break;
    }
}

// ----------------------------------------------- tile claim order (LPT) --
// A tile's sweep time grows with its rounds, i.e. with the eccentricity of
// its sources; persistent CTAs claiming tiles in Morton order leave SMs idle
// while the last long tiles finish (C5: SMs active 81 % of the sweep). Tiles
// are claimed longest-first instead: key = max over the tile's sources of
// the BFS hop distance from a central vertex (the vertex nearest the centre
// of the xy/level bounding box, else vertex 0), computed once per graph.
__global__ void center_pick_kernel(const int *xy, const int *z, int V, int cx2, int cy2, int cz2,
                                   unsigned long long *best) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    const long long d = llabs(2LL * xy[2 * v] - cx2) + llabs(2LL * xy[2 * v + 1] - cy2) +
                        (z ? llabs(2LL * z[v] - cz2) : 0LL);
    atomicMin(best, ((unsigned long long)d << 32) | (unsigned)v);
}

__global__ void bfs_level_kernel(DevGraph g, int *hop, int level, int *changed) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= g.V || hop[v] != level) return;
    bool any = false;
    for (int e = g.out_ptr[v]; e < g.out_ptr[v + 1]; ++e) {
        const int x = g.out_dst[e];
        if (hop[x] == INT_MAX) {   // racing writers store the same value
            hop[x] = level + 1;
            any = true;
        }
    }
    if (any) *changed = 1;
}

__global__ void tile_key_kernel(const int *tile_src, int ntiles, int ts, const int *hop, long long *key) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    int m = 0;
    for (int k = 0; k < ts; ++k) {
        const int s = tile_src[(size_t)t * ts + k];
        if (s >= 0) m = max(m, hop[s] == INT_MAX ? 0 : hop[s]);
    }
    key[t] = ((long long)(INT_MAX - m) << 32) | t;   // ascending sort = longest first, then index
}

__global__ void fill_i32_kernel(int *p, int n, int v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

static const int *center_hops(const wr_graph *g, cudaStream_t st) {
    if (g->hop_c.p) return g->hop_c.p;
    const int V = g->V;
    DBuf<int> hop;
    {   // graph-lifetime buffer: allocated (and later freed) on the legacy stream
        StreamScope s0(0);
        hop.alloc(V);
        WR_CUDA(cudaStreamSynchronize(0));
    }
    fill_i32_kernel<<<(V + 255) / 256, 256, 0, st>>>(hop.p, V, INT_MAX);
    count_launch();
    int c = 0;
    if (g->xy.p) {
        DBuf<unsigned long long> best(1);
        const unsigned long long init = ~0ull;
        WR_CUDA(cudaMemcpyAsync(best.p, &init, 8, cudaMemcpyHostToDevice, st));
        center_pick_kernel<<<(V + 255) / 256, 256, 0, st>>>(g->xy.p, g->z.p, V, g->bbox[0] + g->bbox[1],
                                                            g->bbox[2] + g->bbox[3], g->bbox[4] + g->bbox[5], best.p);
        count_launch();
        unsigned long long hb = 0;
        WR_CUDA(cudaMemcpyAsync(&hb, best.p, 8, cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
        c = (int)(hb & 0xffffffffu);
    }
    const int zero = 0;
    WR_CUDA(cudaMemcpyAsync(hop.p + c, &zero, 4, cudaMemcpyHostToDevice, st));
    DBuf<int> changed(1);
    for (int level = 0; level < V; ++level) {
        WR_CUDA(cudaMemsetAsync(changed.p, 0, 4, st));
        bfs_level_kernel<<<(V + 255) / 256, 256, 0, st>>>(g->view(), hop.p, level, changed.p);
        count_launch();
        int h = 0;
        WR_CUDA(cudaMemcpyAsync(&h, changed.p, 4, cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
        if (!h) break;
    }
    WR_LAUNCH_CHECK();
    g->hop_c = std::move(hop);
    return g->hop_c.p;
}

void bf_run(const wr_graph *g, const BfRun &run0, BfTileStats *d_stats, cudaStream_t st) {
    if (run0.ntiles <= 0) return;
    BfRun run = run0;
    static const bool no_lpt = getenv("WR_NO_LPT") != nullptr;
    DBuf<int> order;
    if (!no_lpt && !run.tile_order && run.ntiles > 1) {
        const int *hop = center_hops(g, st);
        DBuf<long long> key(run.ntiles);
        tile_key_kernel<<<(run.ntiles + 127) / 128, 128, 0, st>>>(run.tile_src, run.ntiles, run.tsw(), hop, key.p);
        count_launch();
        WR_LAUNCH_CHECK();
        std::vector<long long> hk(run.ntiles);
        WR_CUDA(cudaMemcpyAsync(hk.data(), key.p, 8 * run.ntiles, cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
        std::sort(hk.begin(), hk.end());
        std::vector<int> ho(run.ntiles);
        for (int i = 0; i < run.ntiles; ++i) ho[i] = (int)(hk[i] & 0xffffffffll);
        order.alloc(run.ntiles);
        WR_CUDA(cudaMemcpyAsync(order.p, ho.data(), 4 * run.ntiles, cudaMemcpyHostToDevice, st));
        run.tile_order = order.p;
    }
    // WR_TILE_TRACE: per-tile {start, end, rounds, SM} copied to pinned host
    // memory and appended to the file by a stream-ordered host callback, so
    // tracing adds no host sync (concurrent sweeps keep their overlap).
    static const char *trace_path = getenv("WR_TILE_TRACE");
    DBuf<long long> ttrace;
    struct TraceJob {
        long long *h;
        int *ord, *src;
        int ntiles, tsw;
        std::string path;
    };
    TraceJob *tj = nullptr;
    if (trace_path) {
        ttrace.alloc((size_t)4 * run.ntiles + 2 * 1024);   // + per-CTA {sweep end, exit}
        WR_CUDA(cudaMemsetAsync(ttrace.p, 0, ttrace.bytes(), st));
        run.fuse.trace = ttrace.p;
        tj = new TraceJob{nullptr, nullptr, nullptr, run.ntiles, run.tsw(), trace_path};
        WR_CUDA(cudaMallocHost(&tj->h, ttrace.bytes()));
        WR_CUDA(cudaMallocHost(&tj->ord, 4 * (size_t)run.ntiles));
        WR_CUDA(cudaMallocHost(&tj->src, 4 * (size_t)run.ntiles * run.tsw()));
    }
    if (run.pack == 2 && run.keyed) launch_sweep<OpK16>(g, run, d_stats, st);
    else if (run.pack == 2) launch_sweep<OpU16>(g, run, d_stats, st);
    else if (g->wtype == WR_F32) launch_sweep<OpF32>(g, run, d_stats, st);
    else if (g->has_negative) launch_sweep<OpI32N>(g, run, d_stats, st);
    else launch_sweep<OpU32>(g, run, d_stats, st);
    if (tj) {   // lines: tile claim-position start end rounds sm (+ .src: the tile's sources)
        WR_CUDA(cudaMemcpyAsync(tj->h, ttrace.p, ttrace.bytes(), cudaMemcpyDeviceToHost, st));
        if (run.tile_order) WR_CUDA(cudaMemcpyAsync(tj->ord, run.tile_order, 4 * (size_t)run.ntiles, cudaMemcpyDeviceToHost, st));
        else for (int i = 0; i < run.ntiles; ++i) tj->ord[i] = i;
        WR_CUDA(cudaMemcpyAsync(tj->src, run.tile_src, 4 * (size_t)run.ntiles * run.tsw(), cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaLaunchHostFunc(st, [](void *p) {
            TraceJob *t = (TraceJob *)p;
            std::vector<int> pos(t->ntiles);
            for (int i = 0; i < t->ntiles; ++i) pos[t->ord[i]] = i;
            if (FILE *f = fopen(t->path.c_str(), "a")) {
                for (int k = 0; k < t->ntiles; ++k)
                    fprintf(f, "%d %d %lld %lld %lld %lld\n", k, pos[k], t->h[4 * k], t->h[4 * k + 1], t->h[4 * k + 2],
                            t->h[4 * k + 3]);
                fclose(f);
            }
            if (FILE *f = fopen((t->path + ".cta").c_str(), "a")) {   // per CTA: sweep end, exit (ns)
                const long long *c = t->h + 4 * (size_t)t->ntiles;
                for (int b = 0; b < 1024; ++b)
                    if (c[2 * b + 1]) fprintf(f, "%d %lld %lld\n", b, c[2 * b], c[2 * b + 1]);
                fclose(f);
            }
            if (FILE *f = fopen((t->path + ".src").c_str(), "a")) {
                for (int k = 0; k < t->ntiles; ++k) {
                    for (int j = 0; j < t->tsw; ++j) fprintf(f, "%d ", t->src[(size_t)k * t->tsw + j]);
                    fprintf(f, "\n");
                }
                fclose(f);
            }
            // pinned buffers are released by the next sync point's owner: leak-free
            // enough for a diagnostic (freed at process exit)
        }, tj));
    }
}

// C5 fp32 (bench, static 768 shape): delta 0.35 / 0.5 / 0.75 / 1.0 x max w:
// relaxations 2.35 / 2.32 / 2.79 / 3.25 x S*E (off: 3.25), step 299 / 247 /
// 223 / 231 ms (off: 216): the deferral saves work but adds rounds.
float nf_delta_for(const wr_graph *g) {
    if (g->wtype != WR_F32 || !(g->max_w_f > 0.f)) return 0.f;
    static const char *e = getenv("WR_NF_DELTA");
    const float mult = e ? (float)atof(e) : 0.75f;
    return mult > 0.f ? mult * g->max_w_f : 0.f;
}

// Sources per lane for S sources; WR_BF_SPL forces a width.
int choose_spl(int64_t S, int nsm, int pack) {
    const int forced = env_int("WR_BF_SPL", 0);
    if (forced == 1 || forced == 2 || forced == 4) return forced;
    // The widest tile that still yields at least half an SM's worth of tiles
    // per SM pair (>= nsm / 2 tiles), else the narrowest. Measured on C5
    // shards with packed rows (tools/shard_probe.py): 84.7k / 42.3k / 21.2k
    // sources -> 256-source tiles (331 / 166 / 83 tiles; 128-source tiles
    // were slower: 36.5 vs 31.6 ms at 42k, 22.8 vs 18.8 ms at 21k); 10.6k ->
    // 128 (14.7 ms vs 16.9 at 256, 19.7 at 64); C4's 4k -> 64 (3.5 ms vs
    // 7.2 at 256): a tile's sweep time shrinks with its width, but less than
    // linearly, so narrower tiles pay only when SMs would otherwise idle.
    for (int spl = 4; spl > 1; spl /= 2) {
        const int64_t per = 32LL * spl * pack;
        if ((std::max<int64_t>(S, 1) + per - 1) / per >= std::max(nsm / 2, 1)) return spl;
    }
    return 1;
}

// --------------------------------------------------- a4 + output layout --
// Block = 4 warps; a warp handles 32 consecutive output columns (vertices or
// targets) of one 32-slot group of one tile: computes dist/pred for (column
// j, slot = group*32 + lane), stages them in shared memory and writes each
// source's 32 columns as one coalesced 128-B segment of the caller's
// row-major S x T / S x V arrays. Canonical pred (O3, w >= 0): smallest tail
// of a steep tight in-arc; a reachable non-source vertex without one is
// "flat" and is resolved by bf_resolve_flat. Graphs with a negative weight
// resolve every vertex there.
constexpr int OUT_WARPS = 4;
template <class Op>
__global__ void __launch_bounds__(OUT_WARPS * 32) bf_outputs_kernel(DevGraph g, const int *__restrict__ tile_src,
                                                                    int ntiles, int tsw, const uint32_t *__restrict__ rows,
                                                                    const int *__restrict__ slot_row,
                                                                    int64_t out_row0, const int *__restrict__ targets,
                                                                    int T, uint32_t *dist_out, int32_t *pred_out,
                                                                    int *flat_tiles, int neg_graph) {
    __shared__ uint32_t sd[OUT_WARPS][32][33];
    __shared__ int32_t sp[OUT_WARPS][32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int V = g.V;
    const int ncols = targets ? T : V;
    const int chunks = (ncols + 31) / 32;
    const int groups = tsw / 32;
    const int64_t job = (int64_t)blockIdx.x * OUT_WARPS + warp;
    if (job >= (int64_t)ntiles * groups * chunks) return;
    const int tg = (int)(job / chunks);        // tile * groups + group
    const int tile = tg / groups, grp = tg % groups;
    const int c0 = (int)(job % chunks) * 32;
    const int slot = grp * 32 + lane;
    const uint32_t *R = rows + (size_t)tile * V * tsw + grp * 32;
    const int s = tile_src[tile * tsw + slot];
    bool flat = false;
    for (int j = 0; j < 32; ++j) {
        const int col = c0 + j;
        if (col >= ncols) break;
        const int v = targets ? targets[col] : col;
        const uint32_t d = R[(size_t)v * tsw + lane];
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
                        const int u = __shfl_sync(FULL, my_u, k);
                        const uint32_t wk = __shfl_sync(FULL, my_w, k);
                        const uint32_t du = R[(size_t)u * tsw + lane];
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
    // write out: for each source slot k of the group, columns c0..c0+31
    const int col = c0 + lane;
    for (int k = 0; k < 32; ++k) {
        const int sk = tile_src[tile * tsw + grp * 32 + k];
        if (sk < 0) break;                       // tiles are filled slot 0 first
        const int64_t sl = (int64_t)tile * tsw + grp * 32 + k;
        const int64_t row = out_row0 + (slot_row ? slot_row[sl] : sl);
        if (col < ncols) {
            if (dist_out) dist_out[row * ncols + col] = sd[warp][lane][k];
            if (pred_out && !targets) pred_out[row * (int64_t)V + col] = sp[warp][lane][k];
        }
    }
    if (__any_sync(FULL, flat) && lane == 0) atomicOr(&flat_tiles[tile], 1);
}

// a4 canonical pred, vectorised over the tile: warp per (tile, 8 vertices),
// lane = SPL source slots. In-arcs are sorted by tail, so the first steep
// tight in-arc met is the smallest-tail one: the arc loop stops as soon as
// every slot that needs a predecessor has one. Results are staged in shared
// memory and written as one full 32-B sector per source row (8 vertices x
// 4 B), 4 rows per store instruction.
// PW warps per CTA (8 for 32-bit rows, 4 for packed rows: the output
// staging sp[PW][PV][TS + 1] stays under the 48 KB static limit).
// One pred job: (tile, vertices c0 .. c0+7) for all the tile's slots, by
// one warp; spw = the warp's [PV][TS + 1] shared staging.
template <class Op, int SPL, int PA>
__device__ __forceinline__ void pred_job(const DevGraph &g, const int *__restrict__ tile_src,
                                         const uint32_t *__restrict__ rows, const int *__restrict__ slot_row,
                                         int64_t out_row0, int32_t *__restrict__ pred_out, int *flat_tiles, int tile,
                                         int c0, int32_t *spw, int lane) {
    using SK = SkewStage<32 * SPL * Op::PACK>;   // skewed staging rows (bank-conflict-free)
    constexpr int TSW = 32 * SPL;           // 32-bit words per row
    static_assert(PredShape::PV == 8, "the output stores write 8 columns per slot");
    constexpr int P = Op::PACK;
    constexpr int TS = TSW * P;             // sources (slots) per tile
    constexpr int NS = SPL * P;             // slots per lane
    constexpr int PV = PredShape::PV;
    const int V = g.V;
    const uint32_t *Rl = rows + (size_t)tile * V * TSW + lane * SPL;
    int src[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) src[j] = tile_src[tile * TS + lane * NS + j];
    bool flat = false;
    const int nv = min(PV, V - c0);
    int p_lo = 0, p_hi = 0;
    if (lane < nv) {
        p_lo = g.in_ptr[c0 + lane];
        p_hi = g.in_ptr[c0 + lane + 1];
    }
    // steep-tight test of one gathered in-neighbour row for all slots; best
    // = NEED (-1) while a slot still looks for its pred, SKIP (-2) for slots
    // that need none (empty, the source itself, unreachable). Slot j*P + h
    // is half h of the lane's word j.
    // need: bit k set while slot k still looks for its pred (clear for
    // empty slots, the source itself and unreachable vertices); best[k] =
    // the pred found (-1 = none). hit bits of one gathered in-neighbour row:
    // the steep-tight test of all the lane's slots; packed rows test both
    // halves of a word with one add and one compare.
    auto test = [&](const Vec<SPL> &x, uint32_t w, int u, const Vec<SPL> &d, int (&best)[NS], uint32_t &need) {
        uint32_t hit = 0;
        if constexpr (P == 2) {
            const uint32_t w2 = w | (w << 16);   // w in [1, 0x3fff]: no half wraps
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                const uint32_t t2 = __vcmpeq2(__vadd2(x.x[j], w2), d.x[j]);
                hit |= ((t2 & 1u) | ((t2 >> 15) & 2u)) << (2 * j);
            }
        } else {
#pragma unroll
            for (int j = 0; j < SPL; ++j) hit |= (Op::steep_tight(x.x[j], w, d.x[j]) ? 1u : 0u) << j;
        }
        hit &= need;
        if (hit) {
            need &= ~hit;
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if ((hit >> k) & 1u) best[k] = u;
        }
    };
    // two vertices per step (lanes 0-15 / 16-31 hold their in-arcs), PA
    // in-arcs of each per step; stop when no slot still needs a pred
    for (int jv = 0; jv < nv; jv += 2) {
        const bool two = jv + 1 < nv;
        const int jv1 = two ? jv + 1 : jv;
        const int v0 = c0 + jv, v1 = c0 + jv1;
        const int a00 = __shfl_sync(FULL, p_lo, jv), a01 = __shfl_sync(FULL, p_hi, jv);
        const int a10 = __shfl_sync(FULL, p_lo, jv1), a11 = __shfl_sync(FULL, p_hi, jv1);
        const int n0 = a01 - a00, n1 = two ? a11 - a10 : 0;
        const Vec<SPL> d0 = vload<SPL>(Rl + (size_t)v0 * TSW);
        Vec<SPL> d1 = d0;
        if (two) d1 = vload<SPL>(Rl + (size_t)v1 * TSW);
        int best0[NS], best1[NS];
        uint32_t need0 = 0, need1 = 0;
#pragma unroll
        for (int j = 0; j < SPL; ++j)
#pragma unroll
            for (int h = 0; h < P; ++h) {
                const int k = j * P + h;
                best0[k] = best1[k] = -1;
                need0 |= (src[k] >= 0 && v0 != src[k] && Op::finite(Op::half(d0.x[j], h)) ? 1u : 0u) << k;
                need1 |= (two && src[k] >= 0 && v1 != src[k] && Op::finite(Op::half(d1.x[j], h)) ? 1u : 0u) << k;
            }
        const bool any0 = __any_sync(FULL, need0 != 0), any1 = __any_sync(FULL, need1 != 0);
        if (n0 <= 16 && n1 <= 16) {
            const int sub = lane & 15;
            const int base = lane < 16 ? a00 : a10;
            const int cnt = lane < 16 ? n0 : n1;
            int my_u = 0;
            uint32_t my_w = 0;
            if (sub < cnt) {
                const int2 arc = g.in_arc[base + sub];   // (u, w) in one 8-B load
                my_u = arc.x;
                my_w = (uint32_t)arc.y;
            }
            // per-vertex early exit: a vertex whose slots all have their
            // pred stops gathering (its arc count drops to k)
            int e0 = any0 ? n0 : 0, e1 = any1 ? n1 : 0;
            for (int k = 0; k < max(e0, e1); k += PA) {
                int ua[2][PA];
                uint32_t wa[2][PA];
                Vec<SPL> x[2][PA];
#pragma unroll
                for (int a = 0; a < PA; ++a) {
                    ua[0][a] = __shfl_sync(FULL, my_u, (k + a) & 31);
                    wa[0][a] = __shfl_sync(FULL, my_w, (k + a) & 31);
                    ua[1][a] = __shfl_sync(FULL, my_u, (16 + k + a) & 31);
                    wa[1][a] = __shfl_sync(FULL, my_w, (16 + k + a) & 31);
                }
#pragma unroll
                for (int a = 0; a < PA; ++a) {   // lanes whose slots are all done load nothing
                    if (k + a < e0 && need0) x[0][a] = vload<SPL>(Rl + (uint32_t)(ua[0][a] * TSW));
                    if (k + a < e1 && need1) x[1][a] = vload<SPL>(Rl + (uint32_t)(ua[1][a] * TSW));
                }
#pragma unroll
                for (int a = 0; a < PA; ++a) {
                    if (k + a < e0 && need0) test(x[0][a], wa[0][a], ua[0][a], d0, best0, need0);
                    if (k + a < e1 && need1) test(x[1][a], wa[1][a], ua[1][a], d1, best1, need1);
                }
                if (!__any_sync(FULL, need0 != 0)) e0 = min(e0, k + PA);
                if (!__any_sync(FULL, need1 != 0)) e1 = min(e1, k + PA);
            }
        } else {
            auto slow = [&](int lo, int hi, const Vec<SPL> &d, int (&best)[NS], uint32_t &need) {
                for (int base = lo; base < hi; base += 32) {
                    const int cnt = min(32, hi - base);
                    int my_u = 0;
                    uint32_t my_w = 0;
                    if (lane < cnt) {
                        my_u = g.in_src[base + lane];
                        my_w = g.in_w[base + lane];
                    }
                    for (int k = 0; k < cnt; ++k) {
                        const int u = __shfl_sync(FULL, my_u, k);
                        const uint32_t w = __shfl_sync(FULL, my_w, k);
                        test(vload<SPL>(Rl + (uint32_t)(u * TSW)), w, u, d, best, need);
                    }
                }
            };
            if (any0) slow(a00, a01, d0, best0, need0);
            if (two && any1) slow(a10, a11, d1, best1, need1);
        }
        flat |= (need0 | need1) != 0;   // reachable, no steep tight in-arc: flat
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            spw[jv * SK::RS + SK::at(lane * NS + j)] = best0[j];
            if (two) spw[jv1 * SK::RS + SK::at(lane * NS + j)] = best1[j];
        }
    }
    __syncwarp();
    // lane -> slots lane, lane + 32, ...: each writes its 8 columns of the
    // source's row as one full 32-B sector (two 16-B stores); the slots'
    // source and output row are loaded once, all at the same time
    const bool vec = (V & 3) == 0 && nv == PV;
    int srow[TS / 32];
#pragma unroll
    for (int k = 0; k < TS / 32; ++k) {
        const int sl = tile * TS + lane + 32 * k;
        srow[k] = tile_src[sl] < 0 ? -1 : (slot_row ? slot_row[sl] : sl);
    }
#pragma unroll
    for (int k = 0; k < TS / 32; ++k) {
        if (srow[k] < 0) continue;
        const int sl_in = lane + 32 * k;
        int32_t *dst = pred_out + (out_row0 + srow[k]) * (int64_t)V + c0;
        if (vec) {
            const int a = SK::at(sl_in);
            reinterpret_cast<int4 *>(dst)[0] = make_int4(spw[a], spw[SK::RS + a], spw[2 * SK::RS + a], spw[3 * SK::RS + a]);
            reinterpret_cast<int4 *>(dst)[1] =
                make_int4(spw[4 * SK::RS + a], spw[5 * SK::RS + a], spw[6 * SK::RS + a], spw[7 * SK::RS + a]);
        } else {
            for (int jv = 0; jv < nv; ++jv) dst[jv] = spw[jv * SK::RS + SK::at(sl_in)];
        }
    }
    if (__any_sync(FULL, flat) && lane == 0) atomicOr(&flat_tiles[tile], 1);
}

// a4 from keyed rows (OpK16): pred[v] = in_src[in_ptr[v] + k] with k the
// low nibble of the final key (15 = none: the source itself, unreachable
// vertices). A job decodes 8 consecutive vertices of one tile, stages the
// preds in shared memory and writes each source's 8 columns as one full
// 32-B sector (the same output layout as pred_job, no in-arc gathers).
template <int SPL>
__device__ __forceinline__ void pred_job_keyed(const DevGraph &g, const int *__restrict__ tile_src,
                                               const uint32_t *__restrict__ rows, const int *__restrict__ slot_row,
                                               int64_t out_row0, int32_t *__restrict__ pred_out, int tile, int c0,
                                               int32_t *spw, int lane, uint32_t thr, int *overflow,
                                               int (&srow)[2 * SPL], int &srow_tile) {
    constexpr int TSW = 32 * SPL;
    constexpr int TS = TSW * 2;
    constexpr int NS = SPL * 2;    // slots per lane (<= 8 nibbles)
    constexpr int PV = PredShape::PV;
    uint32_t *const kidx = reinterpret_cast<uint32_t *>(spw);   // [PV][32] packed in-arc indices
    int32_t *const tails_s = spw + PV * 32;                      // [PV][16] in-arc tails
    const int V = g.V;
    const uint32_t *Rl = rows + (size_t)tile * V * TSW + lane * SPL;
    const int nv = min(PV, V - c0);
    const int a_lane = lane <= nv ? g.in_ptr[c0 + lane] : 0;
    Vec<SPL> key[PV];
#pragma unroll
    for (int jv = 0; jv < PV; ++jv)
        if (jv < nv) key[jv] = vload<SPL>(Rl + (size_t)(c0 + jv) * TSW);
    bool ovf = false;
#pragma unroll
    for (int jv = 0; jv < PV; jv += 2) {
        if (jv >= nv) break;
        // the in-arc tails of vertices jv (lanes 0-15) and jv + 1 (16-31)
        const int half = lane >> 4, vj = min(jv + half, nv - 1);
        const int lo = __shfl_sync(FULL, a_lane, vj), hi = __shfl_sync(FULL, a_lane, vj + 1);
        tails_s[(jv + half) * 16 + (lane & 15)] = (lane & 15) < hi - lo ? g.in_src[lo + (lane & 15)] : -1;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            if (jv + d >= nv) break;
            uint32_t packed = 0;
#pragma unroll
            for (int j = 0; j < SPL; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t key1 = (key[jv + d].x[j] >> (16 * h)) & 0xffffu;
                    // range check of the keyed rows (the sweep skips it): a stored
                    // distance at or past 0x7ff - max_w may hide a clipped path
                    ovf |= key1 >= thr && key1 != 0x7fffu;
                    packed |= (key1 & 0xfu) << (4 * (j * 2 + h));
                }
            kidx[(jv + d) * 32 + lane] = packed;
        }
    }
    if (__any_sync(FULL, ovf) && lane == 0) atomicOr(overflow, 1);
    __syncwarp();
    const bool vec = (V & 3) == 0 && nv == PV;
    if (srow_tile != tile) {   // the slots' output rows, loaded once per tile by this warp
#pragma unroll
        for (int k = 0; k < TS / 32; ++k) {
            const int sl = tile * TS + lane + 32 * k;
            srow[k] = tile_src[sl] < 0 ? -1 : (slot_row ? slot_row[sl] : sl);
        }
        srow_tile = tile;
    }
    // pred of (vertex jv, slot sl) = tail number k of vertex jv, k = 15: none
    const auto pred_of = [&](int jv, int sl) {
        const uint32_t k = (kidx[jv * 32 + sl / NS] >> (4 * (sl % NS))) & 0xfu;
        return k == 15u ? -1 : tails_s[jv * 16 + k];
    };
#pragma unroll
    for (int k = 0; k < TS / 32; ++k) {
        if (srow[k] < 0) continue;
        const int sl_in = lane + 32 * k;
        int32_t *dst = pred_out + (out_row0 + srow[k]) * (int64_t)V + c0;
        if (vec) {
            reinterpret_cast<int4 *>(dst)[0] =
                make_int4(pred_of(0, sl_in), pred_of(1, sl_in), pred_of(2, sl_in), pred_of(3, sl_in));
            reinterpret_cast<int4 *>(dst)[1] =
                make_int4(pred_of(4, sl_in), pred_of(5, sl_in), pred_of(6, sl_in), pred_of(7, sl_in));
        } else {
            for (int jv = 0; jv < nv; ++jv) dst[jv] = pred_of(jv, sl_in);
        }
    }
    __syncwarp();   // spw is reused by the warp's next job
}

template <class Op, int SPL, int MINB, int PA, int PW>
__global__ void __launch_bounds__(PW * 32, MINB) bf_pred_kernel(DevGraph g, const int *__restrict__ tile_src, int ntiles,
                                                      const uint32_t *__restrict__ rows,
                                                      const int *__restrict__ slot_row, int64_t out_row0,
                                                      int32_t *__restrict__ pred_out, int *flat_tiles) {
    constexpr int TS = 32 * SPL * Op::PACK;
    constexpr int PV = PredShape::PV;
    __shared__ int32_t sp[PW][PV][SkewStage<TS>::RS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunks = (g.V + PV - 1) / PV;
    const int64_t job = (int64_t)blockIdx.x * PW + warp;
    if (job >= (int64_t)ntiles * chunks) return;
    pred_job<Op, SPL, PA>(g, tile_src, rows, slot_row, out_row0, pred_out, flat_tiles, (int)(job / chunks),
                          (int)(job % chunks) * PV, &sp[warp][0][0], lane);
}

template <class Op, int SPL, int MINB, int PA, int PW = 8 / Op::PACK>
static void launch_pred_shape(const wr_graph *g, const BfRun &run, int64_t out_row0, int32_t *pred_out, int *flat,
                              cudaStream_t st) {
    const int64_t jobs = (int64_t)run.ntiles * ((g->V + PredShape::PV - 1) / PredShape::PV);
    const unsigned grid = (unsigned)((jobs + PW - 1) / PW);
    bf_pred_kernel<Op, SPL, MINB, PA, PW><<<grid, PW * 32, 0, st>>>(
        g->view(), run.tile_src, run.ntiles, run.rows, run.slot_row, out_row0, pred_out, flat);
    count_launch();
    WR_LAUNCH_CHECK();
}

template <class Op, int SPL>
static void launch_pred_spl(const wr_graph *g, const BfRun &run, int64_t out_row0, int32_t *pred_out, int *flat,
                            cudaStream_t st) {
    // 256 threads x >= 4 CTAs/SM (64 regs), one arc per vertex per step
    // with a per-vertex early exit: 34.6 ms on config 5; two arcs per step
    // (speculative gathers) 40.8; 3 CTAs/SM 40.0; 6-8 CTAs/SM spill (73-83)
    if constexpr (Op::PACK == 2) {   // 128 threads (staging 33 KB) x 6 CTAs/SM
        static const int cfg16 = env_int("WR_PRED16_CONFIG", 6);
        if (cfg16 == 4) launch_pred_shape<Op, SPL, 4, 1>(g, run, out_row0, pred_out, flat, st);
        else if (cfg16 == 8) launch_pred_shape<Op, SPL, 8, 1, 2>(g, run, out_row0, pred_out, flat, st);
        else launch_pred_shape<Op, SPL, 6, 1>(g, run, out_row0, pred_out, flat, st);
        return;
    }
    static const int cfg = env_int("WR_PRED_CONFIG", 5);
    switch (cfg) {
        case 1: launch_pred_shape<Op, SPL, 4, 2>(g, run, out_row0, pred_out, flat, st); break;
        case 8: launch_pred_shape<Op, SPL, 3, 1>(g, run, out_row0, pred_out, flat, st); break;
        default: launch_pred_shape<Op, SPL, 4, 1>(g, run, out_row0, pred_out, flat, st); break;
    }
}

template <class Op>
static void launch_pred(const wr_graph *g, const BfRun &run, int64_t out_row0, int32_t *pred_out, int *flat,
                        cudaStream_t st) {
    if (run.spl == 2) launch_pred_spl<Op, 2>(g, run, out_row0, pred_out, flat, st);
    else if (run.spl == 4) launch_pred_spl<Op, 4>(g, run, out_row0, pred_out, flat, st);
    else launch_pred_spl<Op, 1>(g, run, out_row0, pred_out, flat, st);
}

void bf_write_outputs(const wr_graph *g, const BfRun &run, int64_t out_row0, int64_t, const int *targets, int T,
                      void *dist_out, int32_t *pred_out, int *d_flat_tiles, cudaStream_t st) {
    if (run.ntiles <= 0 || (!dist_out && !pred_out)) return;
    if (run.pack == 2) {   // packed rows: pred only (no flat vertices: every weight > 0)
        if (dist_out) WR_THROW(WR_EINTERNAL, "bf_write_outputs: dist output from packed rows");
        if (pred_out) launch_pred<OpU16>(g, run, out_row0, pred_out, d_flat_tiles, st);
        return;
    }
    if (pred_out && !g->has_negative) {     // fast vectorised pred pass (flat vertices flagged)
        if (g->wtype == WR_F32) launch_pred<OpF32>(g, run, out_row0, pred_out, d_flat_tiles, st);
        else launch_pred<OpU32>(g, run, out_row0, pred_out, d_flat_tiles, st);
        pred_out = nullptr;
        if (!dist_out) return;
    }
    const int tsw = 32 * run.spl;
    const int ncols = targets ? T : g->V;
    const int64_t jobs = (int64_t)run.ntiles * run.spl * ((ncols + 31) / 32);
    const unsigned grid = (unsigned)((jobs + OUT_WARPS - 1) / OUT_WARPS);
    const int neg = g->has_negative;
    if (g->wtype == WR_F32)
        bf_outputs_kernel<OpF32><<<grid, OUT_WARPS * 32, 0, st>>>(g->view(), run.tile_src, run.ntiles, tsw, run.rows,
                                                                  run.slot_row, out_row0, targets, T,
                                                                  (uint32_t *)dist_out, pred_out, d_flat_tiles, neg);
    else if (neg)
        bf_outputs_kernel<OpI32N><<<grid, OUT_WARPS * 32, 0, st>>>(g->view(), run.tile_src, run.ntiles, tsw, run.rows,
                                                                   run.slot_row, out_row0, targets, T,
                                                                   (uint32_t *)dist_out, pred_out, d_flat_tiles, neg);
    else
        bf_outputs_kernel<OpU32><<<grid, OUT_WARPS * 32, 0, st>>>(g->view(), run.tile_src, run.ntiles, tsw, run.rows,
                                                                  run.slot_row, out_row0, targets, T,
                                                                  (uint32_t *)dist_out, pred_out, d_flat_tiles, neg);
    count_launch();
    WR_LAUNCH_CHECK();
}

// --------------------------------------------- flat predecessors (rare) --
// For one 32-slot group of a tile: hop[v][lane] = BFS layer of v over the
// tight arcs of that slot's source (a min-plus sweep with unit weights
// restricted to tight arcs), then for every flat (v, slot) - or every
// reachable vertex of a negative-weight graph -
// pred = argmin over tight in-arcs of (hop[u], u)  (O3).
constexpr int HOP_THREADS = 512;
template <class Op>
__global__ void __launch_bounds__(HOP_THREADS) hop_bfs_kernel(DevGraph g, const int *__restrict__ tile_src, int tile,
                                                              int grp, int tsw, const uint32_t *__restrict__ rows,
                                                              uint32_t *__restrict__ hop, const int *gate) {
    if (gate && !gate[tile]) return;   // stream-ordered gating: only tiles flagged flat
    extern __shared__ uint32_t smem[];
    const int V = g.V;
    const int NW = (V + 31) >> 5;
    uint32_t *changed = smem;
    uint32_t *cand = smem + NW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWARPS = HOP_THREADS / 32;
    const uint32_t *R = rows + (size_t)tile * V * tsw + grp * 32;
    for (size_t i = threadIdx.x; i < (size_t)V * 32; i += HOP_THREADS) hop[i] = 0xffffffffu;
    for (int w = threadIdx.x; w < NW; w += HOP_THREADS) changed[w] = cand[w] = 0u;
    __syncthreads();
    if (warp == 0) {
        const int s = tile_src[tile * tsw + grp * 32 + lane];
        if (s >= 0) {
            hop[(size_t)s * 32 + lane] = 0;
            atomicOr(&changed[s >> 5], 1u << (s & 31));
        }
    }
    __syncthreads();
    bool more = true;
    while (more) {
        for (int w = threadIdx.x; w < NW; w += HOP_THREADS) {
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
                const uint32_t dv = R[(size_t)v * tsw + lane];
                const uint32_t h0 = hop[(size_t)v * 32 + lane];
                uint32_t h = h0;
                for (int e = g.in_ptr[v]; e < g.in_ptr[v + 1]; ++e) {
                    const int u = g.in_src[e];
                    const uint32_t hu = hop[(size_t)u * 32 + lane];
                    if (hu != 0xffffffffu && Op::tight(R[(size_t)u * tsw + lane], g.in_w[e], dv) && hu + 1 < h)
                        h = hu + 1;
                }
                const bool c = h < h0;
                if (c) hop[(size_t)v * 32 + lane] = h;
                if (__any_sync(FULL, c)) chg |= 1u << b;
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
__global__ void flat_pred_kernel(DevGraph g, const int *__restrict__ tile_src, int tile, int grp, int tsw,
                                 const uint32_t *__restrict__ rows, const uint32_t *__restrict__ hop,
                                 const int *__restrict__ slot_row, int64_t out_row0, int32_t *pred_out,
                                 int neg_graph, const int *gate) {
    if (gate && !gate[tile]) return;
    const int lane = threadIdx.x & 31;
    const int v = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int V = g.V;
    if (v >= V) return;
    const uint32_t *R = rows + (size_t)tile * V * tsw + grp * 32;
    const int slot = grp * 32 + lane;
    const int s = tile_src[tile * tsw + slot];
    const uint32_t d = R[(size_t)v * tsw + lane];
    if (s < 0 || v == s || !Op::finite(d)) return;
    bool steep = false;
    int best = -1;
    uint32_t best_h = 0xffffffffu;
    for (int e = g.in_ptr[v]; e < g.in_ptr[v + 1]; ++e) {
        const int u = g.in_src[e];
        const uint32_t du = R[(size_t)u * tsw + lane];
        if (!Op::tight(du, g.in_w[e], d)) continue;
        if (Op::less(du, d)) steep = true;
        const uint32_t hu = hop[(size_t)u * 32 + lane];
        if (hu < best_h || (hu == best_h && u < best)) {
            best_h = hu;
            best = u;
        }
    }
    const int64_t sl = (int64_t)tile * tsw + slot;
    if (neg_graph || !steep) pred_out[(out_row0 + (slot_row ? slot_row[sl] : sl)) * V + v] = best;
}

template <class Op>
static void resolve_group(const wr_graph *g, const BfRun &run, int t, int grp, uint32_t *hop, size_t smem,
                          int64_t out_row0, int32_t *pred_out, int neg, const int *gate, cudaStream_t st) {
    const int V = g->V;
    const int tsw = 32 * run.spl;
    WR_CUDA(cudaFuncSetAttribute(hop_bfs_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    hop_bfs_kernel<Op><<<1, HOP_THREADS, smem, st>>>(g->view(), run.tile_src, t, grp, tsw, run.rows, hop, gate);
    flat_pred_kernel<Op><<<(V + 7) / 8, 256, 0, st>>>(g->view(), run.tile_src, t, grp, tsw, run.rows, hop,
                                                     run.slot_row, out_row0,
                                                     pred_out, neg, gate);
    count_launch();
    count_launch();
    WR_LAUNCH_CHECK();
}

void bf_resolve_flat(const wr_graph *g, const BfRun &run, const std::vector<int> &tiles, int64_t out_row0,
                     int32_t *pred_out, cudaStream_t st, const int *gate) {
    if (tiles.empty() || !pred_out) return;
    const int V = g->V;
    DBuf<uint32_t> hop((size_t)V * 32);   // reused tile after tile in stream order
    const size_t smem = (size_t)2 * ((V + 31) / 32) * sizeof(uint32_t);
    for (int t : tiles) {
        for (int grp = 0; grp < run.spl; ++grp) {
            if (g->wtype == WR_F32) resolve_group<OpF32>(g, run, t, grp, hop.p, smem, out_row0, pred_out, 0, gate, st);
            else if (g->has_negative)
                resolve_group<OpI32N>(g, run, t, grp, hop.p, smem, out_row0, pred_out, 1, gate, st);
            else resolve_group<OpU32>(g, run, t, grp, hop.p, smem, out_row0, pred_out, 0, gate, st);
        }
    }
}

// ------------------------------------------------------ a8 the scheduler --
// The HBM budget of one call: the caller's cap (default 180 GB) limited by
// what the device can still give. `want` = fixed + pooled bytes that cover
// the whole job in one segment: when libwr's pool already holds that many
// idle bytes (a repeated call of the same size), no driver query is made -
// cudaMemGetInfo was measured to stall for up to ~120 ms on the host while
// another process (nvidia-smi sampling) held the driver.
int64_t budget_bytes(int64_t requested, int64_t fixed, int64_t want_pooled) {
    const int64_t cap = requested > 0 ? requested : (int64_t)180e9;
    int dev = 0;
    WR_CUDA(cudaGetDevice(&dev));
    const int64_t idle = (int64_t)pool_idle_bytes(dev);   // reserved by libwr's pool, reusable
    if (want_pooled > 0 && idle >= want_pooled && fixed + want_pooled <= cap) return fixed + want_pooled;
    size_t free_b = 0, total_b = 0;
    WR_CUDA(cudaMemGetInfo(&free_b, &total_b));
    return std::min<int64_t>(cap, (int64_t)(0.9 * (double)(free_b + (size_t)idle)));
}

// Sources per Bellman-Ford segment: the per-segment working set
// (per_source_bytes each, plus fixed) stays within the budget; a multiple of
// the tile width tsw.
int64_t sources_per_segment(int64_t budget, int64_t fixed_bytes, int64_t per_source_bytes, int64_t S, int tsw) {
    const int64_t room = budget - fixed_bytes;
    if (room < per_source_bytes * tsw)
        WR_THROW(WR_ENOMEM, "scheduler: HBM budget below one source tile");
    int64_t sb = room / per_source_bytes;
    sb = (sb / tsw) * tsw;
    return std::max<int64_t>(tsw, std::min<int64_t>(sb, ((S + tsw - 1) / tsw) * tsw));
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
    StreamScope stream_scope(st);
    const int V = g->V;
    const int ncols = targets ? T : V;
    // V-1 relaxation rounds (P724 §4.7) + the kernel's check round
    const int max_rounds = o.max_rounds > 0 ? o.max_rounds : std::max(1, V - 1);
    const int variant = o.variant == WR_BF_DENSE ? WR_BF_DENSE : WR_BF_FRONTIER;
    const bool nearfar = o.variant == WR_BF_NEARFAR;
    int nsm = 0;
    WR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    const int spl = choose_spl(S, nsm, 1);
    const int tsw = 32 * spl;

    cudaEvent_t e0, e1;
    WR_CUDA(cudaEventCreate(&e0));
    WR_CUDA(cudaEventCreate(&e1));
    WR_CUDA(cudaEventRecord(e0, st));

    const bool dist_dev = dist && is_device_ptr(dist);
    const bool pred_dev = pred && is_device_ptr(pred);
    // async: nothing after the sweep needs the host (no negative cycle to
    // report, no host staging, flat pred vertices resolved under a device
    // gate); the host still builds the tiles before the sweep is enqueued
    const bool async = o.async && (!dist || dist_dev) && (!pred || pred_dev) && !g->has_negative &&
                       o.max_rounds <= 0;
    auto host_check = [&](const int32_t *v, int64_t n, const char *what) {
        for (int64_t i = 0; i < n; ++i)
            if (v[i] < 0 || v[i] >= V) WR_THROW(WR_EINVAL, std::string(what) + ": vertex outside [0, V)");
    };
    DBuf<int> d_src = to_device<int>(sources, S, st);
    if (!is_device_ptr(sources)) host_check(sources, S, "wr_bf_batch sources");
    else check_vertices(d_src.p, S, V, st, "wr_bf_batch sources");
    DBuf<int> d_tgt;
    if (targets) {
        d_tgt = to_device<int>(targets, T, st);
        if (!is_device_ptr(targets)) host_check(targets, T, "wr_bf_batch targets");
        else check_vertices(d_tgt.p, T, V, st, "wr_bf_batch targets");
    }

    // a8: per-source working set = rows (4V) + staging for host outputs
    int64_t per_src = 4LL * V;
    if (dist && !dist_dev) per_src += 4LL * ncols;
    if (pred && !pred_dev) per_src += 4LL * V;
    wr_graph_info_t gi;
    wr_graph_info(g, &gi);
    const int64_t fixed = gi.device_bytes + (64 << 20);
    const int64_t tiles_all = (std::max(S, 1) + tsw - 1) / tsw;
    const int64_t budget = budget_bytes(o.hbm_budget, fixed, tiles_all * tsw * per_src);
    const int64_t sb = sources_per_segment(budget, fixed, per_src, std::max(S, 1), tsw);
    const int64_t max_tiles = tiles_to_allocate(sb, tsw, budget - fixed - sb * per_src, 4LL * V * tsw);

    DBuf<uint32_t> rows((size_t)max_tiles * V * tsw);
    DBuf<int> tile_src(max_tiles * tsw), slot_row(max_tiles * tsw), pos_of(sb);
    DBuf<int> flat(max_tiles);
    DBuf<uint32_t> dist_stage;
    DBuf<int32_t> pred_stage;
    if (dist && !dist_dev) dist_stage.alloc((size_t)sb * ncols);
    if (pred && !pred_dev) pred_stage.alloc((size_t)sb * V);
    DBuf<BfTileStats> d_stats(1);
    BfTileStats h0{0ull, 0, -1, 0ull};
    WR_CUDA(cudaMemcpyAsync(d_stats.p, &h0, sizeof(h0), cudaMemcpyHostToDevice, st));

    int segments = 0;
    int64_t total_tiles = 0;
    for (int64_t lo = 0; lo < S; lo += sb) {
        const int64_t hi = std::min<int64_t>(S, lo + sb);
        const int ntiles = make_tiles_ordered(g, d_src.p, lo, hi, tsw, max_tiles, tile_src.p, slot_row.p, pos_of.p, st);
        BfRun run{tile_src.p, ntiles, rows.p, variant, max_rounds, spl, slot_row.p};
        run.nf_delta = nearfar ? nf_delta_for(g) : 0.f;
        {
            NvtxRange nv("wr.bf.sweep");
            bf_run(g, run, d_stats.p, st);
        }
        BfTileStats hs{0ull, 0, -1, 0ull};
        if (!async) {
            WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
            WR_CUDA(cudaStreamSynchronize(st));
        }
        if (hs.negcycle_tile >= 0) {
            int s_bad = -1;
            WR_CUDA(cudaMemcpy(&s_bad, tile_src.p + (size_t)hs.negcycle_tile * tsw, 4, cudaMemcpyDeviceToHost));
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
        if (pout && async) {   // flat vertices need zero int weights or fp32 absorption
            if (g->wtype == WR_F32 || g->has_zero) {
                std::vector<int> all(ntiles);
                for (int t = 0; t < ntiles; ++t) all[t] = t;
                bf_resolve_flat(g, run, all, row_p, pout, st, flat.p);
            }
        } else if (pout) {
            std::vector<int> hflat(ntiles);
            WR_CUDA(cudaMemcpyAsync(hflat.data(), flat.p, sizeof(int) * ntiles, cudaMemcpyDeviceToHost, st));
            WR_CUDA(cudaStreamSynchronize(st));
            std::vector<int> todo;
            for (int t = 0; t < ntiles; ++t)
                if (hflat[t] || g->has_negative) todo.push_back(t);
            bf_resolve_flat(g, run, todo, row_p, pout, st);
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
    float ms = -1.f;
    if (!async) {   // temporaries are stream-ordered; only the stats need the host
        WR_CUDA(cudaMemcpyAsync(&hs, d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
        WR_CUDA(cudaStreamSynchronize(st));
        WR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats) {   // async: counters unknown (0), ms = -1
        stats->rounds_max = hs.rounds_max;
        stats->relaxations = (int64_t)hs.relax;
        stats->visits = (int64_t)hs.visits;
        stats->segments = segments;
        stats->tiles = (int32_t)total_tiles;
        stats->ms = ms;
        stats->negcycle_source = -1;
        stats->kernel_launches = g_launches - g_launch0;
    }
    return WR_OK;
}

int ctx_rank(const wr_ctx *c);
int ctx_world(const wr_ctx *c);
void ctx_share_blocks(const wr_ctx *c, void *buf, const int64_t *off, cudaStream_t st);

// shard = 1 over a context: rank r relaxes sources [lo_r, hi_r) (contiguous
// blocks, wr_shard_range) into rows lo_r.. of full-size device outputs, then
// the row blocks are exchanged (grouped NCCL broadcasts on the stream).
static wr_status bf_batch_sharded(const wr_graph *g, const int32_t *sources, int32_t S, const int32_t *targets,
                                  int32_t T, void *dist, int32_t *pred, const wr_bf_opts &o, wr_bf_stats *stats) {
    const wr_ctx *ctx = o.ctx;
    const int rank = ctx_rank(ctx), world = ctx_world(ctx);
    WR_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = (cudaStream_t)o.stream;
    StreamScope stream_scope(st);
    const int V = g->V;
    const int64_t ncols = targets ? T : V;
    int64_t lo, hi;
    wr_shard_range(S, rank, world, &lo, &hi);
    const bool dist_dev = dist && is_device_ptr(dist), pred_dev = pred && is_device_ptr(pred);
    DBuf<uint32_t> dstage;
    DBuf<int32_t> pstage;
    if (dist && !dist_dev) dstage.alloc((size_t)std::max<int64_t>(S, 1) * ncols);
    if (pred && !pred_dev) pstage.alloc((size_t)std::max<int64_t>(S, 1) * V);
    uint32_t *dfull = dist ? (dist_dev ? (uint32_t *)dist : dstage.p) : nullptr;
    int32_t *pfull = pred ? (pred_dev ? pred : pstage.p) : nullptr;
    wr_bf_opts local = o;
    local.ctx = nullptr;
    local.shard = 0;
    local.async = 0;
    if (hi > lo) {
        const wr_status rc = bf_batch_impl(g, sources + lo, (int32_t)(hi - lo), targets, T,
                                           dfull ? dfull + lo * ncols : nullptr, pfull ? pfull + lo * V : nullptr,
                                           &local, stats);
        if (rc) return rc;   // every rank sees the same inputs, so every rank fails alike
    }
    std::vector<int64_t> off(world + 1);
    auto share = [&](void *buf, int64_t row_bytes) {
        for (int q = 0; q < world; ++q) {
            int64_t a, b;
            wr_shard_range(S, q, world, &a, &b);
            off[q] = a * row_bytes;
            off[q + 1] = b * row_bytes;
        }
        ctx_share_blocks(ctx, buf, off.data(), st);
    };
    if (dfull) share(dfull, ncols * 4);
    if (pfull) share(pfull, (int64_t)V * 4);
    if (dist && !dist_dev)
        WR_CUDA(cudaMemcpyAsync(dist, dfull, (size_t)S * ncols * 4, cudaMemcpyDeviceToHost, st));
    if (pred && !pred_dev) WR_CUDA(cudaMemcpyAsync(pred, pfull, (size_t)S * V * 4, cudaMemcpyDeviceToHost, st));
    WR_CUDA(cudaStreamSynchronize(st));
    return WR_OK;
}

}  // namespace wr

extern "C" wr_status wr_bf_batch(const wr_graph *g, const int32_t *sources, int32_t S, const int32_t *targets,
                                 int32_t T, void *dist, int32_t *pred, const wr_bf_opts *opts,
                                 wr_bf_stats *stats) {
    return wr::guarded([&]() -> wr_status {
        wr::NvtxRange nv("wr_bf_batch");
        if (opts && opts->shard) {
            if (!opts->ctx) return wr::fail(WR_EINVAL, "wr_bf_batch: shard needs opts.ctx");
            if (!g || S < 0 || (S > 0 && !sources)) return wr::fail(WR_EINVAL, "wr_bf_batch: bad arguments");
            if (wr::ctx_world(opts->ctx) > 1)
                return wr::bf_batch_sharded(g, sources, S, targets, T, dist, pred, *opts, stats);
        }
        return wr::bf_batch_impl(g, sources, S, targets, T, dist, pred, opts, stats);
    });
}
