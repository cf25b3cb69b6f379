/*
 * wr_oracle.c - the plain, slow, obviously-correct CPU oracle for the
 * warehouse-routing hot path of arXiv:2504.20655.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2504_20655_b200/csrc); neither side includes or links the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC -pthread
 *   (no FMA contraction, no FTZ/DAZ: every fp32 add is one IEEE-754
 *    binary32 round-to-nearest-even addition, SSE2 on x86-64).
 *
 * Citations: P<line> = /root/reference/PAPER.md line, with its section;
 * S<line> = SPEC.md line; O<k>/A<k> = the readings listed in DESIGN.md
 * (taken from SURVEY.md §8(c)).
 *
 * Functions and what pins them (tests/test_oracle_*.py):
 *   orc_bf            O2 Bellman-Ford (P720-724 §4.7)  pinned: Dijkstra, FW,
 *                     closed forms (grid Manhattan, aisle formula), 3-aisle
 *                     worked example, negative-cycle fixtures.
 *   orc_pred          O3 canonical predecessor          pinned: V1-V4 validity
 *                     predicate + brute-force tie cases of the worked example.
 *   orc_route_cost    O4 left-to-right route cost (P658 §4.6) pinned: worked
 *                     example D, hand sums.
 *   orc_exact_route   O5 exhaustive lexicographic search (P658 §4.6, P322 §3)
 *                     pinned: independent Held-Karp (cost + argmin for int),
 *                     120-cost histogram of the worked example.
 *   orc_exact_route_range  O6 rank-range chunk (P658 §4.6)  pinned: chunked ==
 *                     unchunked, SPEC plan_segmentation examples.
 *   orc_segmented_route  O7 Theorem 3.1 stitch (P324-337 §3) pinned: worked
 *                     example labelings, m=1 == exact, singletons == exact,
 *                     segmented >= exact, candidate counts vs Thm 3.1.
 *   orc_segmented_pairs_route  NEXT-1 boundary-pair stitch:
 *                     pinned: m=1 == exact, singletons == exact, and for int
 *                     weights == (min cost, lex-smallest) over ALL segment-
 *                     contiguous orders by brute force; int cost <= O7's.
 *   orc_held_karp_route  NEXT-2 exact route for 13-16 stops (subset DP +
 *                     backward feasibility + lexicographic greedy, P370 §3)
 *                     pinned: == itertools brute force (cost, order, rank) on
 *                     n <= 8 fp32 absorption matrices and the committed
 *                     reproducers (tests/golden/hk_absorption.txt); == O5 on
 *                     n <= 9 incl. tie-heavy matrices; cost == the tests'
 *                     independent Python Held-Karp for n up to 13.
 *   orc_closed_route_cost / orc_exact_closed_route / orc_held_karp_closed_route
 *   / orc_segmented_closed_route / orc_segmented_pairs_closed_route
 *                     NEXT-4 closed tour through a depot (reading R4, P320 §3:
 *                     the paper leaves entrance/exit out; the closed variant
 *                     adds the two depot legs) pinned: hand-checked tour of the
 *                     3-aisle example (cost 32, rank 1, 8 optima); itertools
 *                     brute force (cost, rank, order) incl. fp32 absorption;
 *                     zero legs == every open counterpart bit for bit;
 *                     singletons == exact; pairs == brute force over
 *                     segment-contiguous closed orders (int).
 *   orc_kmeans        O8 deterministic integer K-means   pinned: hand-made
 *                     separated clusters, brute-force Lloyd fixpoint check.
 *   orc_order_stops   a2 stop projection (P226-238 §2.4) pinned: numpy unique.
 *   orc_route_orders  a2..a7 composed (per order), threads over sources/orders.
 *   orc_certificate   P9 fixpoint certificate for full-size GPU outputs.
 *   orc_pred_certificate  P9 from pred rows alone (rebuilt path sums) + the
 *                     O3 canonical rule; pinned: oracle rows pass, mutated
 *                     rows (non-canonical tie, non-arc, cycle, dropped
 *                     vertex, wrong root) fail.
 *   orc_pred_many     O3 on many rows (threads only).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_I32 0
#define ORC_F32 1

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2
#define ORC_ENEGCYCLE 3
#define ORC_EOVERFLOW 4
#define ORC_EUNREACHABLE 5
#define ORC_ETOOLARGE 6

#define I32_INF INT32_MAX

/* ------------------------------------------------------------------------ */
/* O2  Bellman-Ford, textbook Gauss-Seidel form over the COO arcs in file     */
/* order (P720-724 §4.7: "(V-1) relaxation rounds"; S385-393 bellman_ford).   */
/* Early exit when a round changes nothing (reading A9: dist is identical).   */
/* int weights: d in int64, INF = INT32_MAX; fp32: d[s] = +0.0f, INF = +inf,  */
/* c = d[u] + w is one binary32 addition.                                     */
/* Returns ORC_ENEGCYCLE if after V-1 rounds an arc still relaxes.            */
/* ------------------------------------------------------------------------ */
int orc_bf(int V, long long E, const int *src, const int *dst, const void *w,
           int wtype, int s, void *dist_out, int *rounds_out)
{
    if (V <= 0 || s < 0 || s >= V) return ORC_EINVAL;
    int rounds = 0;
    if (wtype == ORC_I32) {
        const int *wi = (const int *)w;
        int64_t *d = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
        if (!d) return ORC_ENOMEM;
        for (int v = 0; v < V; ++v) d[v] = I32_INF;
        d[s] = 0;
        int changed = 1;
        for (int round = 1; round <= V - 1 && changed; ++round) {
            changed = 0;
            for (long long e = 0; e < E; ++e) {
                int u = src[e], v = dst[e];
                if (d[u] == I32_INF) continue;
                int64_t c = d[u] + (int64_t)wi[e];
                if (c < d[v]) { d[v] = c; changed = 1; }
            }
            if (changed) rounds = round;
        }
        if (changed) { /* V-1 rounds used up: one more pass decides */
            for (long long e = 0; e < E; ++e) {
                int u = src[e], v = dst[e];
                if (d[u] == I32_INF) continue;
                if (d[u] + (int64_t)wi[e] < d[v]) { free(d); return ORC_ENEGCYCLE; }
            }
        }
        int *out = (int *)dist_out;
        for (int v = 0; v < V; ++v) out[v] = (int)d[v];
        free(d);
    } else {
        const float *wf = (const float *)w;
        float *d = (float *)dist_out;
        for (int v = 0; v < V; ++v) d[v] = INFINITY;
        d[s] = 0.0f;
        int changed = 1;
        for (int round = 1; round <= V - 1 && changed; ++round) {
            changed = 0;
            for (long long e = 0; e < E; ++e) {
                int u = src[e], v = dst[e];
                if (isinf(d[u])) continue;
                float c = d[u] + wf[e];
                if (c < d[v]) { d[v] = c; changed = 1; }
            }
            if (changed) rounds = round;
        }
        /* fp32 weights are finite and >= 0 (reading A8): no negative cycle. */
    }
    if (rounds_out) *rounds_out = rounds;
    return ORC_OK;
}

/* tight(u->v) <=> d[u] finite and fl(d[u]+w) == d[v] (exactly / bitwise).   */
static int tight_arc(int wtype, const void *dist, const void *w, long long e,
                     int u, int v)
{
    if (wtype == ORC_I32) {
        const int *d = (const int *)dist;
        if (d[u] == I32_INF) return 0;
        return (int64_t)d[u] + (int64_t)((const int *)w)[e] == (int64_t)d[v];
    } else {
        const float *d = (const float *)dist;
        if (isinf(d[u])) return 0;
        float c = d[u] + ((const float *)w)[e];
        return c == d[v];
    }
}

static int finite_at(int wtype, const void *dist, int v)
{
    if (wtype == ORC_I32) return ((const int *)dist)[v] != I32_INF;
    return !isinf(((const float *)dist)[v]);
}

static int less_at(int wtype, const void *dist, int a, int b) /* d[a] < d[b] */
{
    if (wtype == ORC_I32) return ((const int *)dist)[a] < ((const int *)dist)[b];
    return ((const float *)dist)[a] < ((const float *)dist)[b];
}

/* ------------------------------------------------------------------------ */
/* O3  Canonical predecessor (reading A5; the paper is silent, P721 §4.7 only */
/* says pred is V x N). Depends on dist alone, so it is schedule-free.        */
/*   any negative weight in the graph (int only):                             */
/*       pred[v] = argmin over tight in-arcs (u->v) of (hop[u], u)            */
/*   else (all weights >= 0):                                                 */
/*       steep = {u : tight(u->v), d[u] < d[v]}; pred[v] = min steep if any,  */
/*       else ("flat" v) argmin over tight in-arcs of (hop[u], u)             */
/*   hop = BFS layer over tight arcs from s; pred[s] = -1; unreachable -1.    */
/* ------------------------------------------------------------------------ */
int orc_pred(int V, long long E, const int *src, const int *dst, const void *w,
             int wtype, int s, const void *dist, int *pred)
{
    int has_neg = 0;
    if (wtype == ORC_I32)
        for (long long e = 0; e < E; ++e) if (((const int *)w)[e] < 0) has_neg = 1;

    int *steep = (int *)malloc(sizeof(int) * (size_t)V);
    int *need_hop = (int *)calloc((size_t)V, sizeof(int));
    if (!steep || !need_hop) { free(steep); free(need_hop); return ORC_ENOMEM; }
    for (int v = 0; v < V; ++v) { steep[v] = -1; pred[v] = -1; }

    for (long long e = 0; e < E; ++e) {
        int u = src[e], v = dst[e];
        if (v == s || !tight_arc(wtype, dist, w, e, u, v)) continue;
        if (!has_neg && less_at(wtype, dist, u, v)) {
            if (steep[v] < 0 || u < steep[v]) steep[v] = u;
        }
    }
    int any_hop = 0;
    for (int v = 0; v < V; ++v) {
        if (v == s || !finite_at(wtype, dist, v)) continue;
        if (steep[v] >= 0) pred[v] = steep[v];
        else { need_hop[v] = 1; any_hop = 1; }
    }
    if (any_hop) {
        /* BFS over the tight arcs from s (adjacency by plain counting sort). */
        int *cnt = (int *)calloc((size_t)V + 1, sizeof(int));
        long long ntight = 0;
        for (long long e = 0; e < E; ++e)
            if (tight_arc(wtype, dist, w, e, src[e], dst[e])) { cnt[src[e] + 1]++; ntight++; }
        for (int v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
        int *adj = (int *)malloc(sizeof(int) * (size_t)(ntight > 0 ? ntight : 1));
        int *fill = (int *)malloc(sizeof(int) * (size_t)V);
        int *hop = (int *)malloc(sizeof(int) * (size_t)V);
        int *queue = (int *)malloc(sizeof(int) * (size_t)V);
        memcpy(fill, cnt, sizeof(int) * (size_t)V);
        for (long long e = 0; e < E; ++e)
            if (tight_arc(wtype, dist, w, e, src[e], dst[e])) adj[fill[src[e]]++] = dst[e];
        for (int v = 0; v < V; ++v) hop[v] = -1;
        int head = 0, tail = 0;
        hop[s] = 0; queue[tail++] = s;
        while (head < tail) {
            int x = queue[head++];
            for (int k = cnt[x]; k < cnt[x + 1]; ++k) {
                int y = adj[k];
                if (hop[y] < 0) { hop[y] = hop[x] + 1; queue[tail++] = y; }
            }
        }
        for (long long e = 0; e < E; ++e) {
            int u = src[e], v = dst[e];
            if (!need_hop[v] || !tight_arc(wtype, dist, w, e, u, v) || hop[u] < 0) continue;
            int p = pred[v];
            if (p < 0 || hop[u] < hop[p] || (hop[u] == hop[p] && u < p)) pred[v] = u;
        }
        free(cnt); free(adj); free(fill); free(hop); free(queue);
    }
    free(steep); free(need_hop);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* O4  Route cost: c_1 = D[p0][p1], c_t = fl(c_{t-1} + D[p_{t-1}][p_t]);      */
/* n = 1 -> 0; any INF leg -> INF. Open route, depot excluded (P322 §3).      */
/* D is directed and never mirrored (reading A15). int sums are exact; a     */
/* finite sum outside int32 -> ORC_EOVERFLOW.                                 */
/* ------------------------------------------------------------------------ */
int orc_route_cost(int wtype, const void *D, int n, const int *seq, int len, void *cost_out)
{
    if (wtype == ORC_I32) {
        const int *Di = (const int *)D;
        int64_t c = 0;
        int inf = 0;
        for (int t = 1; t < len; ++t) {
            int leg = Di[(size_t)seq[t - 1] * n + seq[t]];
            if (leg == I32_INF) inf = 1;
            else c += leg;
        }
        if (inf) { *(int *)cost_out = I32_INF; return ORC_OK; }
        if (c >= I32_INF || c < INT32_MIN) return ORC_EOVERFLOW;
        *(int *)cost_out = (int)c;
    } else {
        const float *Df = (const float *)D;
        float c = 0.0f;
        if (len >= 2) c = Df[(size_t)seq[0] * n + seq[1]];
        for (int t = 2; t < len; ++t) c = c + Df[(size_t)seq[t - 1] * n + seq[t]];
        *(float *)cost_out = c;
    }
    return ORC_OK;
}

/* std::next_permutation in C: lexicographic successor; 0 when wrapped. */
static int next_perm(int *a, int n)
{
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) --i;
    if (i < 0) return 0;
    int j = n - 1;
    while (a[j] <= a[i]) --j;
    int t = a[i]; a[i] = a[j]; a[j] = t;
    for (int l = i + 1, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
    return 1;
}

static long long factorial(int n)
{
    long long f = 1;
    for (int k = 2; k <= n; ++k) f *= k;
    return f;
}

/* Lehmer decode: the permutation of [0,n) with lexicographic rank r. */
static void unrank(long long r, int n, int *perm)
{
    int used[32] = {0};
    for (int k = 0; k < n; ++k) {
        long long f = factorial(n - 1 - k);
        long long q = r / f;
        r %= f;
        for (int x = 0; x < n; ++x) {
            if (used[x]) continue;
            if (q == 0) { perm[k] = x; used[x] = 1; break; }
            --q;
        }
    }
}

/* Lehmer code: lexicographic rank of a permutation of [0,n). */
long long orc_perm_rank(const int *perm, int n)
{
    long long r = 0;
    for (int k = 0; k < n; ++k) {
        int smaller = 0;
        for (int l = k + 1; l < n; ++l) if (perm[l] < perm[k]) ++smaller;
        r += smaller * factorial(n - 1 - k);
    }
    return r;
}

static int cost_less(int wtype, const void *a, const void *b)
{
    if (wtype == ORC_I32) return *(const int *)a < *(const int *)b;
    return *(const float *)a < *(const float *)b;
}

static int cost_equal(int wtype, const void *a, const void *b)
{
    if (wtype == ORC_I32) return *(const int *)a == *(const int *)b;
    return *(const float *)a == *(const float *)b;
}

/* ------------------------------------------------------------------------ */
/* O6  Exhaustive evaluation of the lexicographic rank range [lo, hi)        */
/* (P658 §4.6: "one thread per permutation ... (n-1) transitions";            */
/* "segmenting the computation ... multiple kernel launches").                */
/* Keeps the first minimum (strict <): ties -> smallest rank.                 */
/* ------------------------------------------------------------------------ */
int orc_exact_route_range(int wtype, const void *D, int n, long long lo, long long hi,
                          int *seq_out, void *cost_out, long long *rank_out)
{
    if (n < 1 || n > 20 || lo < 0 || hi > factorial(n) || lo >= hi) return ORC_EINVAL;
    int perm[32];
    unrank(lo, n, perm);
    char best[4] = {0}, cur[4] = {0};
    long long best_rank = -1;
    for (long long r = lo; r < hi; ++r) {
        int rc = orc_route_cost(wtype, D, n, perm, n, cur);
        if (rc) return rc;
        if (best_rank < 0 || cost_less(wtype, cur, best)) {
            memcpy(best, cur, 4);
            best_rank = r;
            memcpy(seq_out, perm, sizeof(int) * (size_t)n);
        }
        if (r + 1 < hi) next_perm(perm, n);
    }
    memcpy(cost_out, best, 4);
    *rank_out = best_rank;
    return ORC_OK;
}

/* O5  Exact route: all n! directed sequences (reading A2), first minimum.   */
int orc_exact_route(int wtype, const void *D, int n, int *seq_out, void *cost_out,
                    long long *rank_out)
{
    return orc_exact_route_range(wtype, D, n, 0, factorial(n), seq_out, cost_out, rank_out);
}

/* ------------------------------------------------------------------------ */
/* NEXT-2 exact route for up to 16 stops by the Held-Karp subset DP (the     */
/* paper mentions Held-Karp O(n^2 2^n) as the exact-TSP alternative, P370   */
/* §3; reading R2 in DESIGN.md). Same result as O5:     */
/* the minimum left-to-right cost over all n! orders, ties -> the           */
/* lexicographically smallest order. Three steps:                           */
/*  1. forward DP over states (S, j) = stop set S visited, ending at j:      */
/*     F({j}, j) = 0, F(S, j) = min over i in S-{j} of fl(F(S-{j}, i) +     */
/*     D[i][j]); C* = min_j F(all, j). fl(c + d) is monotone in c, so the    */
/*     minimum of the left-to-right sums is exact (reading A16).            */
/*  2. backward feasibility: M(S, j) = the largest prefix cost c with which  */
/*     some completion of (S, j) still ends at a cost <= C*:                 */
/*     M(all, j) = C*; M(S, j) = max over k not in S of                     */
/*     inv(D[j][k], M(S+{k}, k)), inv(d, m) = max{c : fl(c + d) <= m}       */
/*     (int: m - d exactly; fp32: bisection over the ordered bit patterns   */
/*     of c >= 0, valid because fl(c + d) is monotone in c); "none" if no c. */
/*  3. lexicographic greedy: the first stop is the smallest a with           */
/*     M({a}, a) >= 0 (prefix cost 0), each next stop the smallest k not    */
/*     yet visited with fl(c + D[j][k]) <= M(S+{k}, k). No order costs less  */
/*     than C*, so "<= C*" is "== C*": the greedy walks the lexicographically */
/*     smallest optimal order, which is O5's first minimum.                   */
/* Keeping one cheapest prefix per state (the earlier version) is NOT enough */
/* for fp32: fl(c + d) is monotone but not strictly, so a costlier,         */
/* lexicographically smaller prefix can tie after rounding.    */
/* If every order costs INF (an INF leg in each), O5 returns the identity.  */
/* int sums in int64 (INF leg -> INF); a finite result outside int32 ->     */
/* ORC_EOVERFLOW.                                                           */
/* ------------------------------------------------------------------------ */
static float f32_of_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }

/* max{c >= 0 float : fl(c + d) <= m}, or -1 if none (d, m >= 0 or +inf). */
static float f32_inv(float d, float m)
{
    if (!(0.0f + d <= m)) return -1.0f;              /* not even c = 0 */
    uint32_t lo = 0, hi = 0x7f800000u;               /* +0 .. +inf      */
    if (f32_of_bits(hi) + d <= m) return f32_of_bits(hi);
    while (hi - lo > 1) {                            /* P(lo) true, P(hi) false */
        uint32_t mid = lo + (hi - lo) / 2;
        if (f32_of_bits(mid) + d <= m) lo = mid; else hi = mid;
    }
    return f32_of_bits(lo);
}

/* din / dout (NEXT-4 closed tour, reading R4): NULL for the open route, or  */
/* the n depot legs D[depot][j] and D[i][depot]: the tour is depot -> pi ->  */
/* depot, summed left to right from the first depot leg.                     */
static int held_karp_impl(int wtype, const void *D, const void *din, const void *dout, int n,
                          int *seq_out, void *cost_out, long long *rank_out);

int orc_held_karp_route(int wtype, const void *D, int n, int *seq_out, void *cost_out,
                        long long *rank_out)
{
    return held_karp_impl(wtype, D, NULL, NULL, n, seq_out, cost_out, rank_out);
}

static int held_karp_impl(int wtype, const void *D, const void *din, const void *dout, int n,
                          int *seq_out, void *cost_out, long long *rank_out)
{
    if (n < 1 || n > 16) return ORC_EINVAL;
    if (n == 1 && !din) {
        seq_out[0] = 0;
        memset(cost_out, 0, 4);
        *rank_out = 0;
        return ORC_OK;
    }
    const size_t NS = (size_t)1 << n, F = NS - 1;
    const int64_t IINF = INT64_MAX / 4, NONE = INT64_MIN;
    const int *Di = (const int *)D;
    const float *Df = (const float *)D;
    int64_t *ci = NULL;        /* int:  F then M, [S * n + j] */
    float *cf = NULL;          /* fp32: F then M              */
    if (wtype == ORC_I32) ci = (int64_t *)malloc(sizeof(int64_t) * NS * (size_t)n);
    else cf = (float *)malloc(sizeof(float) * NS * (size_t)n);
    if (!ci && !cf) return ORC_ENOMEM;
    /* 1. forward DP */
    for (size_t S = 1; S < NS; ++S) {
        for (int j = 0; j < n; ++j) {
            if (!((S >> j) & 1)) continue;
            const size_t P = S & ~((size_t)1 << j), st = S * n + j;
            if (P == 0) {   /* first stop: prefix cost 0, or the depot leg */
                if (ci) {
                    const int leg = din ? ((const int *)din)[j] : 0;
                    ci[st] = leg == I32_INF ? IINF : leg;
                } else {
                    cf[st] = din ? ((const float *)din)[j] : 0.0f;
                }
                continue;
            }
            int first = 1;
            for (int i = 0; i < n; ++i) {
                if (!((P >> i) & 1)) continue;
                if (ci) {
                    const int leg = Di[(size_t)i * n + j];
                    const int64_t pre = ci[P * n + i];
                    const int64_t c = (leg == I32_INF || pre >= IINF) ? IINF : pre + leg;
                    if (first || c < ci[st]) ci[st] = c;
                } else {
                    const float c = cf[P * n + i] + Df[(size_t)i * n + j];
                    if (first || c < cf[st]) cf[st] = c;
                }
                first = 0;
            }
        }
    }
    int64_t cstar_i = 0;
    float cstar_f = 0.0f;
    for (int j = 0; j < n; ++j) {   /* closed: + the return leg */
        if (ci) {
            int64_t c = ci[F * n + j];
            if (dout) {
                const int leg = ((const int *)dout)[j];
                c = (leg == I32_INF || c >= IINF) ? IINF : c + leg;
            }
            if (j == 0 || c < cstar_i) cstar_i = c;
        } else {
            const float c = dout ? cf[F * n + j] + ((const float *)dout)[j] : cf[F * n + j];
            if (j == 0 || c < cstar_f) cstar_f = c;
        }
    }
    int all_inf = ci ? cstar_i >= IINF : isinf(cstar_f);
    if (all_inf) {                                   /* every order costs INF: O5 keeps rank 0 */
        for (int a = 0; a < n; ++a) seq_out[a] = a;
        if (ci) *(int *)cost_out = I32_INF; else *(float *)cost_out = INFINITY;
        *rank_out = 0;
        free(ci); free(cf);
        return ORC_OK;
    }
    /* 2. backward feasibility bound M (overwrites F, full set first) */
    for (size_t S = NS - 1; S >= 1; --S) {
        for (int j = 0; j < n; ++j) {
            if (!((S >> j) & 1)) continue;
            const size_t st = S * n + j;
            if (S == F) {   /* M(all, j) = C*, or the largest prefix whose return leg stays <= C* */
                if (!dout) { if (ci) ci[st] = cstar_i; else cf[st] = cstar_f; }
                else if (ci) {
                    const int leg = ((const int *)dout)[j];
                    ci[st] = leg == I32_INF ? NONE : cstar_i - leg;
                } else {
                    cf[st] = f32_inv(((const float *)dout)[j], cstar_f);
                }
                continue;
            }
            int64_t bi = NONE;
            float bf = -1.0f;
            for (int k = 0; k < n; ++k) {
                if ((S >> k) & 1) continue;
                const size_t nx = (S | ((size_t)1 << k)) * n + k;
                if (ci) {
                    const int leg = Di[(size_t)j * n + k];
                    if (leg == I32_INF || ci[nx] == NONE) continue;
                    const int64_t c = ci[nx] - leg;      /* max c with c + leg <= M */
                    if (c > bi) bi = c;
                } else {
                    if (cf[nx] < 0.0f) continue;
                    const float c = f32_inv(Df[(size_t)j * n + k], cf[nx]);
                    if (c > bf) bf = c;
                }
            }
            if (ci) ci[st] = bi; else cf[st] = bf;
        }
        if (S == 1) break;
    }
    /* 3. lexicographic greedy along the feasible states */
    size_t S = 0;
    int j = -1;
    int64_t pi = 0;
    float pf = 0.0f;
    for (int t = 0; t < n; ++t) {
        int pick = -1;
        for (int k = 0; k < n && pick < 0; ++k) {
            if ((S >> k) & 1) continue;
            const size_t nx = (S | ((size_t)1 << k)) * n + k;
            if (ci) {
                const int first = din ? ((const int *)din)[k] : 0;
                const int64_t c = t == 0 ? (first == I32_INF ? IINF : first)
                                         : (Di[(size_t)j * n + k] == I32_INF ? IINF : pi + Di[(size_t)j * n + k]);
                if (ci[nx] != NONE && c < IINF && c <= ci[nx]) { pick = k; pi = c; }
            } else {
                const float c = t == 0 ? (din ? ((const float *)din)[k] : 0.0f) : pf + Df[(size_t)j * n + k];
                if (cf[nx] >= 0.0f && c <= cf[nx]) { pick = k; pf = c; }
            }
        }
        if (pick < 0) { free(ci); free(cf); return ORC_EINVAL; }   /* unreachable by construction */
        seq_out[t] = pick;
        S |= (size_t)1 << pick;
        j = pick;
    }
    if (dout) {   /* the return leg */
        if (ci) pi += ((const int *)dout)[j];
        else pf = pf + ((const float *)dout)[j];
    }
    int rc = ORC_OK;
    if (ci) {
        if (pi >= I32_INF || pi < INT32_MIN) rc = ORC_EOVERFLOW;
        else *(int *)cost_out = (int)pi;
    } else {
        *(float *)cost_out = pf;
    }
    *rank_out = orc_perm_rank(seq_out, n);
    free(ci); free(cf);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4 closed tour (reading R4 in DESIGN.md). The    */
/* paper assumes "the entrance and exit are the same in the warehouse, and   */
/* that these are not part of the route" (P320 §3); the closed variant puts  */
/* them back: the picker leaves the depot, visits every stop, and returns.   */
/* cost(pi) = left-to-right sum over the n + 2 legs depot -> pi_0 -> ... ->  */
/* pi_{n-1} -> depot: c = D[dep][pi_0], c = fl(c + D[pi_{t-1}][pi_t]), then  */
/* fl(c + D[pi_{n-1}][dep]). It is O4 on the augmented matrix whose index n */
/* is the depot as the first stop and n + 1 the depot as the last, so the    */
/* arithmetic is O4's. din[j] = D[dep][j], dout[i] = D[i][dep].              */
/* ------------------------------------------------------------------------ */
static void *closed_aug(const void *D, const void *din, const void *dout, int n)
{
    const int m = n + 2;
    char *A = (char *)calloc((size_t)m * m, 4);
    if (!A) return NULL;
    for (int i = 0; i < n; ++i) {
        memcpy(A + 4 * ((size_t)i * m), (const char *)D + 4 * ((size_t)i * n), 4 * (size_t)n);
        memcpy(A + 4 * ((size_t)n * m + i), (const char *)din + 4 * (size_t)i, 4);        /* depot -> i */
        memcpy(A + 4 * ((size_t)i * m + n + 1), (const char *)dout + 4 * (size_t)i, 4);   /* i -> depot */
    }
    return A;
}

static int closed_cost_aug(int wtype, const void *A, int n, const int *seq, int len, void *cost_out)
{
    int aug[40];
    aug[0] = n;
    for (int t = 0; t < len; ++t) aug[t + 1] = seq[t];
    aug[len + 1] = n + 1;
    return orc_route_cost(wtype, A, n + 2, aug, len + 2, cost_out);
}

int orc_closed_route_cost(int wtype, const void *D, const void *din, const void *dout, int n,
                          const int *seq, int len, void *cost_out)
{
    if (n < 1 || n > 32 || len < 0 || len > 32) return ORC_EINVAL;
    void *A = closed_aug(D, din, dout, n);
    if (!A) return ORC_ENOMEM;
    int rc = closed_cost_aug(wtype, A, n, seq, len, cost_out);
    free(A);
    return rc;
}

/* Exact closed tour: all n! orders (std::next_permutation order), first     */
/* minimum (strict <): ties -> the lexicographically smallest order (O5).     */
int orc_exact_closed_route(int wtype, const void *D, const void *din, const void *dout, int n,
                           int *seq_out, void *cost_out, long long *rank_out)
{
    if (n < 1 || n > 12) return ORC_EINVAL;
    void *A = closed_aug(D, din, dout, n);
    if (!A) return ORC_ENOMEM;
    int perm[32];
    for (int k = 0; k < n; ++k) perm[k] = k;
    char best[4] = {0}, cur[4] = {0};
    long long r = 0, best_rank = -1;
    do {
        int rc = closed_cost_aug(wtype, A, n, perm, n, cur);
        if (rc) { free(A); return rc; }
        if (best_rank < 0 || cost_less(wtype, cur, best)) {
            memcpy(best, cur, 4);
            best_rank = r;
            memcpy(seq_out, perm, sizeof(int) * (size_t)n);
        }
        ++r;
    } while (next_perm(perm, n));
    free(A);
    memcpy(cost_out, best, 4);
    *rank_out = best_rank;
    return ORC_OK;
}

/* Held-Karp closed tour for up to 16 stops: the same three steps as         */
/* orc_held_karp_route with the depot legs folded in (first state cost =     */
/* D[dep][j]; C* and the backward bound include the return leg).             */
int orc_held_karp_closed_route(int wtype, const void *D, const void *din, const void *dout, int n,
                               int *seq_out, void *cost_out, long long *rank_out)
{
    return held_karp_impl(wtype, D, din, dout, n, seq_out, cost_out, rank_out);
}

/* O6 combine: chunks of <= C permutations, (cost, rank) lexicographic min. */
int orc_exact_route_chunked(int wtype, const void *D, int n, long long chunk,
                            int *seq_out, void *cost_out, long long *rank_out,
                            long long *nchunks_out)
{
    if (chunk < 1) return ORC_EINVAL;
    long long N = factorial(n), nch = 0, best_rank = -1;
    char best[4] = {0};
    int seq[32];
    for (long long lo = 0; lo < N; lo += chunk) {
        long long hi = lo + chunk < N ? lo + chunk : N;
        char c[4];
        long long r;
        int rc = orc_exact_route_range(wtype, D, n, lo, hi, seq, c, &r);
        if (rc) return rc;
        ++nch;
        if (best_rank < 0 || cost_less(wtype, c, best)
            || (cost_equal(wtype, c, best) && r < best_rank)) {
            memcpy(best, c, 4);
            best_rank = r;
            memcpy(seq_out, seq, sizeof(int) * (size_t)n);
        }
    }
    memcpy(cost_out, best, 4);
    *rank_out = best_rank;
    if (nchunks_out) *nchunks_out = nch;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* O7  Segmented route, Theorem 3.1 (P324-337 §3; P670 §4.6; P816 §6).        */
/* 1. segments = nonempty label groups, relabelled by first appearance over  */
/*    stop index; stops within a segment in ascending index.                 */
/* 2. sigma_j = O5 over the segment's D submatrix; boundary nodes = its      */
/*    first and last stop (P333-334 "two boundary nodes").                   */
/* 3. stitch: every segment order tau (lexicographic) x orientation mask b    */
/*    (bit k reverses the k-th segment in tau order): candidate = the        */
/*    concatenation, cost = full O4 recompute over all n stops (reading A13). */
/* 4. min cost, ties -> lexicographically smallest concatenated sequence.    */
/* counts_out[0] = sum n_j! segment sequences, counts_out[1] = m'! 2^m'      */
/* stitch candidates (twice Thm 3.1's undirected counts, reading A2).        */
/* ------------------------------------------------------------------------ */
static int segmented_impl(int wtype, const void *D, const void *din, const void *dout, int n,
                          const int *labels, int *seq_out, void *cost_out, long long *counts_out);

int orc_segmented_route(int wtype, const void *D, int n, const int *labels,
                        int *seq_out, void *cost_out, long long *counts_out)
{
    return segmented_impl(wtype, D, NULL, NULL, n, labels, seq_out, cost_out, counts_out);
}

/* NEXT-4 (reading R4): O7 for the closed tour - the segments' own routes    */
/* stay open (Theorem 3.1 clusters), the stitch costs each concatenation as  */
/* the full closed tour (depot legs included).                               */
int orc_segmented_closed_route(int wtype, const void *D, const void *din, const void *dout, int n,
                               const int *labels, int *seq_out, void *cost_out, long long *counts_out)
{
    return segmented_impl(wtype, D, din, dout, n, labels, seq_out, cost_out, counts_out);
}

static int segmented_impl(int wtype, const void *D, const void *din, const void *dout, int n,
                          const int *labels, int *seq_out, void *cost_out, long long *counts_out)
{
    if (n < 1 || n > 32) return ORC_EINVAL;
    int seg_of[32], nseg = 0, map_lab[32], map_id[32], nmap = 0;
    for (int i = 0; i < n; ++i) {
        int id = -1;
        for (int k = 0; k < nmap; ++k) if (map_lab[k] == labels[i]) id = map_id[k];
        if (id < 0) { map_lab[nmap] = labels[i]; map_id[nmap] = nseg; id = nseg++; ++nmap; }
        seg_of[i] = id;
    }
    if (nseg > 8) return ORC_ETOOLARGE;
    int seg_len[8] = {0}, seg_stops[8][32], seg_route[8][32];
    for (int i = 0; i < n; ++i) seg_stops[seg_of[i]][seg_len[seg_of[i]]++] = i;
    long long seg_evals = 0;
    size_t esz = 4;
    for (int j = 0; j < nseg; ++j) {
        int nj = seg_len[j];
        if (nj > 12) return ORC_ETOOLARGE;
        char *sub = (char *)malloc(esz * (size_t)nj * (size_t)nj);
        for (int a = 0; a < nj; ++a)
            for (int b = 0; b < nj; ++b)
                memcpy(sub + esz * ((size_t)a * nj + b),
                       (const char *)D + esz * ((size_t)seg_stops[j][a] * n + seg_stops[j][b]), esz);
        int local[32];
        char c[4];
        long long r;
        int rc = orc_exact_route(wtype, sub, nj, local, c, &r);
        free(sub);
        if (rc) return rc;
        for (int a = 0; a < nj; ++a) seg_route[j][a] = seg_stops[j][local[a]];
        seg_evals += factorial(nj);
    }
    int tau[8];
    for (int k = 0; k < nseg; ++k) tau[k] = k;
    int best_seq[32], cand[32], have = 0;
    char best[4] = {0}, cur[4] = {0};
    long long stitched = 0;
    do {
        for (int b = 0; b < (1 << nseg); ++b) {
            int pos = 0;
            for (int k = 0; k < nseg; ++k) {
                int j = tau[k], nj = seg_len[j];
                for (int a = 0; a < nj; ++a)
                    cand[pos++] = ((b >> k) & 1) ? seg_route[j][nj - 1 - a] : seg_route[j][a];
            }
            int rc = din ? orc_closed_route_cost(wtype, D, din, dout, n, cand, n, cur)
                         : orc_route_cost(wtype, D, n, cand, n, cur);
            if (rc) return rc;
            ++stitched;
            int better = !have || cost_less(wtype, cur, best);
            if (!better && cost_equal(wtype, cur, best)) {
                for (int t = 0; t < n; ++t) {
                    if (cand[t] != best_seq[t]) { better = cand[t] < best_seq[t]; break; }
                }
            }
            if (better) { have = 1; memcpy(best, cur, 4); memcpy(best_seq, cand, sizeof(int) * (size_t)n); }
        }
    } while (next_perm(tau, nseg));
    memcpy(seq_out, best_seq, sizeof(int) * (size_t)n);
    memcpy(cost_out, best, 4);
    if (counts_out) { counts_out[0] = seg_evals; counts_out[1] = stitched; }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1 boundary-pair segmented route (reading R1 in  */
/* DESIGN.md). The paper stitches one fixed best route per segment in both  */
/* orientations (O7, P324-337 §3). This variant keeps, per segment, the best */
/* open path for every ordered endpoint pair (first a, last b):             */
/*  1. relabel segments by first appearance (as O7);                         */
/*  2. per segment j (n_j <= 9 stops): enumerate all n_j! orders of its stops */
/*     lexicographically, cost each left to right (O4), and keep for its    */
/*     (first, last) pair the first strictly cheaper order (ties -> the     */
/*     lexicographically smallest); a single stop is its own path;          */
/*  3. stitch: for every segment order (m! of them, lexicographic) and every */
/*     choice of one endpoint pair per segment, concatenate the kept paths, */
/*     cost the full n-stop sequence left to right, keep the minimum, ties  */
/*     -> the lexicographically smallest sequence.                          */
/* Candidates m! * prod_j pairs_j <= 2^26, else ETOOLARGE (as the GPU).      */
/* counts_out = {segment orders evaluated, stitch candidates}.               */
/* ------------------------------------------------------------------------ */
static int pairs_impl(int wtype, const void *D, const void *din, const void *dout, int n, const int *labels,
                      int *seq_out, void *cost_out, long long *counts_out);

int orc_segmented_pairs_route(int wtype, const void *D, int n, const int *labels,
                              int *seq_out, void *cost_out, long long *counts_out)
{
    return pairs_impl(wtype, D, NULL, NULL, n, labels, seq_out, cost_out, counts_out);
}

/* NEXT-4 x NEXT-1: the pair stitch of a closed tour (segment paths open,    */
/* every stitch candidate costed as the full closed tour).                   */
int orc_segmented_pairs_closed_route(int wtype, const void *D, const void *din, const void *dout, int n,
                                     const int *labels, int *seq_out, void *cost_out, long long *counts_out)
{
    return pairs_impl(wtype, D, din, dout, n, labels, seq_out, cost_out, counts_out);
}

static int pairs_impl(int wtype, const void *D, const void *din, const void *dout, int n, const int *labels,
                      int *seq_out, void *cost_out, long long *counts_out)
{
    if (n < 1 || n > 16) return ORC_EINVAL;
    int seg_of[16], nseg = 0, map_lab[16], map_id[16], nmap = 0;
    for (int i = 0; i < n; ++i) {
        int id = -1;
        for (int k = 0; k < nmap; ++k) if (map_lab[k] == labels[i]) id = map_id[k];
        if (id < 0) { map_lab[nmap] = labels[i]; map_id[nmap] = nseg; id = nseg++; ++nmap; }
        seg_of[i] = id;
    }
    if (nseg > 6) return ORC_ETOOLARGE;
    int seg_len[6] = {0}, seg_stops[6][16];
    for (int i = 0; i < n; ++i) seg_stops[seg_of[i]][seg_len[seg_of[i]]++] = i;
    /* step 2: best path per (segment, first, last); path[j][a][b][0..nj) */
    static __thread int path[6][9][9][9];
    static __thread char pcost[6][9][9][4];
    static __thread int have[6][9][9];
    long long seg_evals = 0;
    int npairs[6], pair_a[6][81], pair_b[6][81];
    for (int j = 0; j < nseg; ++j) {
        const int nj = seg_len[j];
        if (nj > 9) return ORC_ETOOLARGE;
        memset(have[j], 0, sizeof(have[j]));
        int loc[9], g[9];
        for (int a = 0; a < nj; ++a) loc[a] = a;
        do {
            for (int a = 0; a < nj; ++a) g[a] = seg_stops[j][loc[a]];
            char c[4] = {0};
            if (nj >= 2) {
                int rc = orc_route_cost(wtype, D, n, g, nj, c);
                if (rc) return rc;
            }
            ++seg_evals;
            const int fa = loc[0], lb = loc[nj - 1];
            if (!have[j][fa][lb] || cost_less(wtype, c, pcost[j][fa][lb])) {
                have[j][fa][lb] = 1;
                memcpy(pcost[j][fa][lb], c, 4);
                memcpy(path[j][fa][lb], g, sizeof(int) * (size_t)nj);
            }
        } while (next_perm(loc, nj));
        npairs[j] = 0;
        for (int a = 0; a < nj; ++a)
            for (int b = 0; b < nj; ++b)
                if (have[j][a][b]) { pair_a[j][npairs[j]] = a; pair_b[j][npairs[j]] = b; ++npairs[j]; }
    }
    long long ncand = factorial(nseg);
    for (int j = 0; j < nseg; ++j) ncand *= npairs[j];
    if (ncand > (1ll << 26)) return ORC_ETOOLARGE;
    /* step 3: stitch over segment orders x endpoint pairs, full recompute */
    int tau[6];
    for (int k = 0; k < nseg; ++k) tau[k] = k;
    int best_seq[16], cand[16], got = 0;
    char best[4] = {0}, cur[4] = {0};
    long long stitched = 0;
    do {
        int choice[6] = {0};
        for (;;) {
            int pos = 0;
            for (int k = 0; k < nseg; ++k) {
                const int j = tau[k], nj = seg_len[j];
                const int a = pair_a[j][choice[k]], b = pair_b[j][choice[k]];
                for (int t = 0; t < nj; ++t) cand[pos++] = path[j][a][b][t];
            }
            if (din) {
                int rc = orc_closed_route_cost(wtype, D, din, dout, n, cand, n, cur);
                if (rc) return rc;
            } else if (n >= 2) {
                int rc = orc_route_cost(wtype, D, n, cand, n, cur);
                if (rc) return rc;
            } else {
                memset(cur, 0, 4);
            }
            ++stitched;
            int better = !got || cost_less(wtype, cur, best);
            if (!better && cost_equal(wtype, cur, best)) {
                for (int t = 0; t < n; ++t) {
                    if (cand[t] != best_seq[t]) { better = cand[t] < best_seq[t]; break; }
                }
            }
            if (better) { got = 1; memcpy(best, cur, 4); memcpy(best_seq, cand, sizeof(int) * (size_t)n); }
            /* next endpoint choice: mixed radix, last segment fastest */
            int k = nseg - 1;
            while (k >= 0 && ++choice[k] == npairs[tau[k]]) { choice[k] = 0; --k; }
            if (k < 0) break;
        }
    } while (next_perm(tau, nseg));
    memcpy(seq_out, best_seq, sizeof(int) * (size_t)n);
    memcpy(cost_out, best, 4);
    if (counts_out) { counts_out[0] = seg_evals; counts_out[1] = stitched; }
    return ORC_OK;
}

/* Theorem 3.1 (P326-329 §3): undirected count m! 2^(m-1) + (1/2) sum n_j!,  */
/* and the brute-force undirected count n!/2.                                 */
void orc_route_count_reduction(int m, const int *n_j, unsigned long long *reduced,
                               unsigned long long *brute)
{
    unsigned long long mf = 1, half = 0, n = 0;
    for (int k = 2; k <= m; ++k) mf *= (unsigned long long)k;
    for (int j = 0; j < m; ++j) { half += (unsigned long long)factorial(n_j[j]); n += (unsigned long long)n_j[j]; }
    *reduced = mf * (1ull << (m - 1)) + half / 2;
    *brute = (unsigned long long)factorial((int)n) / 2;
}

/* ------------------------------------------------------------------------ */
/* O8  Deterministic integer K-means segment plan (reading A12; the paper    */
/* clusters stops with K-means, P322 §3, P670 §4.6, init/ties unspecified).   */
/* K = min(K, n). Farthest-point init: c0 = stop 0, next = argmax of min     */
/* squared distance to chosen centres (ties -> smallest index). Lloyd steps: */
/* assign to the rational centroid (Sx/cnt, Sy/cnt) of least squared          */
/* distance, compared cross-multiplied in exact integers, ties -> lower       */
/* cluster; empty cluster keeps its centroid; stop when the assignment       */
/* repeats or after 100 assignments.                                          */
/* ------------------------------------------------------------------------ */
static __int128 sqd_scaled(long long x, long long y, long long sx, long long sy, long long cnt)
{   /* cnt^2 * |p - S/cnt|^2 = (cnt x - Sx)^2 + (cnt y - Sy)^2 */
    __int128 dx = (__int128)cnt * x - sx, dy = (__int128)cnt * y - sy;
    return dx * dx + dy * dy;
}

int orc_kmeans(const int *xy, int n, int K, int *labels)
{
    if (n < 1 || K < 1) return ORC_EINVAL;
    if (K > n) K = n;
    if (K > 32) return ORC_EINVAL;
    int centre[32];
    centre[0] = 0;
    for (int k = 1; k < K; ++k) {
        long long best = -1;
        int arg = 0;
        for (int p = 0; p < n; ++p) {
            long long mind = -1;
            for (int q = 0; q < k; ++q) {
                long long dx = (long long)xy[2 * p] - xy[2 * centre[q]];
                long long dy = (long long)xy[2 * p + 1] - xy[2 * centre[q] + 1];
                long long d = dx * dx + dy * dy;
                if (mind < 0 || d < mind) mind = d;
            }
            if (mind > best) { best = mind; arg = p; }
        }
        centre[k] = arg;
    }
    long long sx[32], sy[32], cnt[32];
    for (int k = 0; k < K; ++k) { sx[k] = xy[2 * centre[k]]; sy[k] = xy[2 * centre[k] + 1]; cnt[k] = 1; }
    int prev[64], have_prev = 0;
    for (int it = 0; it < 100; ++it) {
        for (int p = 0; p < n; ++p) {
            int arg = 0;
            for (int k = 1; k < K; ++k) {
                /* d_k < d_arg  <=>  sqd_k * cnt_arg^2 < sqd_arg * cnt_k^2 */
                __int128 lhs = sqd_scaled(xy[2 * p], xy[2 * p + 1], sx[k], sy[k], cnt[k]) * ((__int128)cnt[arg] * cnt[arg]);
                __int128 rhs = sqd_scaled(xy[2 * p], xy[2 * p + 1], sx[arg], sy[arg], cnt[arg]) * ((__int128)cnt[k] * cnt[k]);
                if (lhs < rhs) arg = k;
            }
            labels[p] = arg;
        }
        if (have_prev && memcmp(prev, labels, sizeof(int) * (size_t)n) == 0) break;
        memcpy(prev, labels, sizeof(int) * (size_t)n);
        have_prev = 1;
        for (int k = 0; k < K; ++k) {
            long long nx = 0, ny = 0, c = 0;
            for (int p = 0; p < n; ++p) if (labels[p] == k) { nx += xy[2 * p]; ny += xy[2 * p + 1]; ++c; }
            if (c > 0) { sx[k] = nx; sy[k] = ny; cnt[k] = c; }
        }
    }
    return ORC_OK;
}

/* a2  Stop projection (P226-238 §2.4): an order's stops are its distinct    */
/* location nodes, sorted ascending. Returns the stop count.                  */
int orc_order_stops(const int *nodes, int count, int *stops)
{
    int n = 0;
    for (int a = 0; a < count; ++a) {
        int x = nodes[a], seen = 0;
        for (int b = 0; b < n; ++b) if (stops[b] == x) seen = 1;
        if (!seen) stops[n++] = x;
    }
    for (int a = 1; a < n; ++a) {           /* insertion sort */
        int x = stops[a], b = a - 1;
        while (b >= 0 && stops[b] > x) { stops[b + 1] = stops[b]; --b; }
        stops[b + 1] = x;
    }
    return n;
}

/* ------------------------------------------------------------------------ */
/* Threaded composition over independent units (sources, then orders).       */
/* ------------------------------------------------------------------------ */
typedef struct {
    int V; long long E; const int *src, *dst; const void *w; int wtype;
    const int *sources; int S; void *rows; int *rc; int next; pthread_mutex_t mu;
} bf_job;

static void *bf_worker(void *arg)
{
    bf_job *j = (bf_job *)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int k = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (k >= j->S) break;
        j->rc[k] = orc_bf(j->V, j->E, j->src, j->dst, j->w, j->wtype, j->sources[k],
                          (char *)j->rows + (size_t)4 * j->V * k, NULL);
    }
    return NULL;
}

/* BF from S sources with nthreads std-thread-style workers; rows S x V. */
int orc_bf_many(int V, long long E, const int *src, const int *dst, const void *w,
                int wtype, const int *sources, int S, void *rows, int nthreads)
{
    bf_job j = {V, E, src, dst, w, wtype, sources, S, rows, NULL, 0, PTHREAD_MUTEX_INITIALIZER};
    j.rc = (int *)calloc((size_t)(S > 0 ? S : 1), sizeof(int));
    if (nthreads < 1) nthreads = 1;
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, bf_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    int rc = ORC_OK;
    for (int k = 0; k < S; ++k) if (j.rc[k]) { rc = j.rc[k]; break; }
    free(j.rc);
    return rc;
}

/* O3 for S rows at once: orc_pred per row on nthreads workers (threading  */
/* only; every row is the plain sequential orc_pred above).                  */
typedef struct {
    int V; long long E; const int *src, *dst; const void *w; int wtype;
    const int *sources; int S; const void *dist; int *pred; int *rc;
    int next; pthread_mutex_t mu;
} pred_job;

static void *pred_worker(void *arg)
{
    pred_job *j = (pred_job *)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int k = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (k >= j->S) break;
        j->rc[k] = orc_pred(j->V, j->E, j->src, j->dst, j->w, j->wtype, j->sources[k],
                            (const char *)j->dist + (size_t)4 * j->V * k, j->pred + (size_t)j->V * k);
    }
    return NULL;
}

int orc_pred_many(int V, long long E, const int *src, const int *dst, const void *w,
                  int wtype, const int *sources, int S, const void *dist, int *pred, int nthreads)
{
    pred_job j = {V, E, src, dst, w, wtype, sources, S, dist, pred, NULL, 0, PTHREAD_MUTEX_INITIALIZER};
    j.rc = (int *)calloc((size_t)(S > 0 ? S : 1), sizeof(int));
    if (!j.rc) return ORC_ENOMEM;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, pred_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    int rc = ORC_OK;
    for (int k = 0; k < S; ++k) if (j.rc[k]) { rc = j.rc[k]; break; }
    free(j.rc);
    return rc;
}

typedef struct {
    int wtype, V; const int *row_of; const void *rows;
    const long long *order_ptr; const int *order_nodes; long long B;
    int m; const int *xy; const int *labels_in;
    int *out_n; int *out_seq; void *out_cost; long long *out_rank; int *out_rc;
    long long next; pthread_mutex_t mu; int pairs; int depot;
} route_job;

static void *route_worker(void *arg)
{
    route_job *j = (route_job *)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        long long o = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (o >= j->B) break;
        long long lo = j->order_ptr[o], hi = j->order_ptr[o + 1];
        int stops[64];
        if (hi - lo > 64) { j->out_rc[o] = ORC_ETOOLARGE; continue; }
        int n = orc_order_stops(j->order_nodes + lo, (int)(hi - lo), stops);
        j->out_n[o] = n;
        if (n > 16) { j->out_rc[o] = ORC_ETOOLARGE; continue; }
        char D[16 * 16 * 4];
        int unreachable = 0;
        for (int a = 0; a < n; ++a) {
            const char *row = (const char *)j->rows + (size_t)4 * j->V * j->row_of[stops[a]];
            for (int b = 0; b < n; ++b) {
                memcpy(D + 4 * (a * n + b), row + 4 * (size_t)stops[b], 4);
                if (!finite_at(j->wtype, row, stops[b])) unreachable = 1;
            }
        }
        /* NEXT-4 closed tour: the depot legs, from the depot's row and the   */
        /* stops' rows at the depot column                                    */
        char din[16 * 4], dout[16 * 4];
        const int closed = j->depot >= 0;
        if (closed) {
            const char *drow = (const char *)j->rows + (size_t)4 * j->V * j->row_of[j->depot];
            for (int a = 0; a < n; ++a) {
                memcpy(din + 4 * a, drow + 4 * (size_t)stops[a], 4);
                const char *row = (const char *)j->rows + (size_t)4 * j->V * j->row_of[stops[a]];
                memcpy(dout + 4 * a, row + 4 * (size_t)j->depot, 4);
                if (!finite_at(j->wtype, drow, stops[a]) || !finite_at(j->wtype, row, j->depot)) unreachable = 1;
            }
        }
        if (unreachable) { j->out_rc[o] = ORC_EUNREACHABLE; continue; }
        int seq[32], rc;
        char cost[4];
        long long rank = 0;
        if (j->m <= 1) {
            if (closed)
                rc = n > 12 ? orc_held_karp_closed_route(j->wtype, D, din, dout, n, seq, cost, &rank)
                            : orc_exact_closed_route(j->wtype, D, din, dout, n, seq, cost, &rank);
            else if (n > 12) rc = orc_held_karp_route(j->wtype, D, n, seq, cost, &rank);   /* NEXT-2 */
            else rc = orc_exact_route(j->wtype, D, n, seq, cost, &rank);
        } else {
            int labels[32], xy[64];
            if (j->labels_in) {
                memcpy(labels, j->labels_in + lo, sizeof(int) * (size_t)n); /* caller: aligned w/ stops */
            } else {
                for (int a = 0; a < n; ++a) { xy[2 * a] = j->xy[2 * stops[a]]; xy[2 * a + 1] = j->xy[2 * stops[a] + 1]; }
                orc_kmeans(xy, n, j->m, labels);
            }
            long long counts[2];
            if (closed && j->pairs) rc = orc_segmented_pairs_closed_route(j->wtype, D, din, dout, n, labels, seq, cost, counts);
            else if (closed) rc = orc_segmented_closed_route(j->wtype, D, din, dout, n, labels, seq, cost, counts);
            else if (j->pairs) rc = orc_segmented_pairs_route(j->wtype, D, n, labels, seq, cost, counts);
            else rc = orc_segmented_route(j->wtype, D, n, labels, seq, cost, counts);
            rank = orc_perm_rank(seq, n);
        }
        j->out_rc[o] = rc;
        if (rc) continue;
        for (int a = 0; a < n; ++a) j->out_seq[o * 16 + a] = stops[seq[a]];
        memcpy((char *)j->out_cost + 4 * o, cost, 4);
        j->out_rank[o] = rank;
    }
    return NULL;
}

/* a2..a7 for a batch of orders: stops -> distinct sources -> BF rows ->      */
/* per-order D -> exact (m <= 1) or segmented (m >= 2, O8 labels from xy;     */
/* pairs != 0: the NEXT-1 boundary-pair stitch) route. out_seq is B x 16 node */
/* ids. Returns the first failing code.                                       */
int orc_route_orders(int V, long long E, const int *src, const int *dst, const void *w,
                     int wtype, const long long *order_ptr, const int *order_nodes,
                     long long B, int m, const int *xy, int nthreads,
                     int *out_n, int *out_seq, void *out_cost, long long *out_rank,
                     int *out_rc, int pairs, int depot)
{
    if (depot >= V) return ORC_EINVAL;
    int *row_of = (int *)malloc(sizeof(int) * (size_t)V);
    for (int v = 0; v < V; ++v) row_of[v] = -1;
    long long L = order_ptr[B];
    for (long long a = 0; a < L; ++a) row_of[order_nodes[a]] = 1;
    if (depot >= 0) row_of[depot] = 1;   /* NEXT-4: the depot is a BF source too */
    int S = 0;
    for (int v = 0; v < V; ++v) if (row_of[v] >= 0) row_of[v] = S++;
    int *sources = (int *)malloc(sizeof(int) * (size_t)(S > 0 ? S : 1));
    for (int v = 0; v < V; ++v) if (row_of[v] >= 0) sources[row_of[v]] = v;
    void *rows = malloc((size_t)4 * V * (size_t)(S > 0 ? S : 1));
    if (!rows) { free(row_of); free(sources); return ORC_ENOMEM; }
    int rc = orc_bf_many(V, E, src, dst, w, wtype, sources, S, rows, nthreads);
    if (rc == ORC_OK) {
        route_job j = {wtype, V, row_of, rows, order_ptr, order_nodes, B, m, xy, NULL,
                       out_n, out_seq, out_cost, out_rank, out_rc, 0, PTHREAD_MUTEX_INITIALIZER, pairs, depot};
        pthread_t th[256];
        if (nthreads < 1) nthreads = 1;
        if (nthreads > 256) nthreads = 256;
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, route_worker, &j);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
        for (long long o = 0; o < B; ++o) if (out_rc[o]) { rc = out_rc[o]; break; }
    }
    free(rows); free(row_of); free(sources);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* P9  Fixpoint certificate (w >= 0 or exact int): dist (S x V) equals the   */
/* oracle's iff (i) d[s] = 0, (ii) every arc has d[v] <= fl(d[u]+w),          */
/* (iii) pred passes V1-V4: pred[s] = -1; d[v] finite <=> pred[v] != -1;     */
/* some arc pred[v]->v is tight; following pred reaches s in <= V-1 steps.   */
/* Returns the number of violating rows (0 = certified).                      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int V; long long E; const int *src, *dst; const void *w; int wtype;
    const int *in_ptr_i; const long long *in_ptr; const int *in_src; const long long *in_arc;
    const int *sources; int S; const void *dist; const int *pred; long long *bad;
    int next; pthread_mutex_t mu;
} cert_job;

static int cert_row(cert_job *j, int k)
{
    int V = j->V, s = j->sources[k];
    const void *d = (const char *)j->dist + (size_t)4 * V * k;
    const int *p = j->pred ? j->pred + (size_t)V * k : NULL;
    if (j->wtype == ORC_I32) { if (((const int *)d)[s] != 0) return 1; }
    else { float z = ((const float *)d)[s]; if (z != 0.0f || signbit(z)) return 1; }
    for (long long e = 0; e < j->E; ++e) {
        int u = j->src[e], v = j->dst[e];
        if (!finite_at(j->wtype, d, u)) continue;
        if (j->wtype == ORC_I32) {
            if ((int64_t)((const int *)d)[u] + ((const int *)j->w)[e] < (int64_t)((const int *)d)[v]) return 2;
        } else {
            float c = ((const float *)d)[u] + ((const float *)j->w)[e];
            if (c < ((const float *)d)[v]) return 2;
        }
    }
    if (!p) return 0;
    if (p[s] != -1) return 3;
    for (int v = 0; v < V; ++v) {
        if (v == s) continue;
        int fin = finite_at(j->wtype, d, v);
        if (fin != (p[v] != -1)) return 4;
        if (!fin) continue;
        int u = p[v], ok = 0;
        if (u < 0 || u >= V) return 5;
        for (long long q = j->in_ptr[v]; q < j->in_ptr[v + 1]; ++q) {
            long long e = j->in_arc[q];
            if (j->src[e] == u && tight_arc(j->wtype, d, j->w, e, u, v)) { ok = 1; break; }
        }
        if (!ok) return 5;
    }
    /* V4: depth along pred, memoised; -2 = on the current walk (cycle). */
    int *depth = (int *)malloc(sizeof(int) * (size_t)V);
    int *stack = (int *)malloc(sizeof(int) * (size_t)V);
    for (int v = 0; v < V; ++v) depth[v] = -1;
    depth[s] = 0;
    int bad = 0;
    for (int v = 0; v < V && !bad; ++v) {
        if (depth[v] >= 0 || p[v] == -1) continue;
        int top = 0, x = v;
        while (depth[x] == -1) { depth[x] = -2; stack[top++] = x; x = p[x]; if (x < 0) { bad = 1; break; } }
        if (bad || depth[x] == -2) { bad = 1; break; }
        int dd = depth[x];
        while (top > 0) { int y = stack[--top]; depth[y] = ++dd; if (dd > V - 1) bad = 1; }
    }
    free(depth); free(stack);
    return bad ? 6 : 0;
}

static void *cert_worker(void *arg)
{
    cert_job *j = (cert_job *)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int k = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (k >= j->S) break;
        int r = cert_row(j, k);
        if (r) __atomic_add_fetch(j->bad, 1, __ATOMIC_RELAXED);
    }
    return NULL;
}

long long orc_certificate(int V, long long E, const int *src, const int *dst, const void *w,
                          int wtype, const int *sources, int S, const void *dist,
                          const int *pred, int nthreads)
{
    long long *in_ptr = (long long *)calloc((size_t)V + 1, sizeof(long long));
    long long *in_arc = (long long *)malloc(sizeof(long long) * (size_t)(E > 0 ? E : 1));
    long long *fill = (long long *)malloc(sizeof(long long) * (size_t)V);
    for (long long e = 0; e < E; ++e) in_ptr[dst[e] + 1]++;
    for (int v = 0; v < V; ++v) in_ptr[v + 1] += in_ptr[v];
    memcpy(fill, in_ptr, sizeof(long long) * (size_t)V);
    for (long long e = 0; e < E; ++e) in_arc[fill[dst[e]]++] = e;
    long long bad = 0;
    cert_job j = {V, E, src, dst, w, wtype, NULL, in_ptr, NULL, in_arc, sources, S, dist, pred,
                  &bad, 0, PTHREAD_MUTEX_INITIALIZER};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, cert_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(in_ptr); free(in_arc); free(fill);
    return bad;
}

/* ------------------------------------------------------------------------ */
/* P9 from pred rows alone (full-size GPU outputs whose dist rows are not    */
/* returned): per row, (a) pred must be a tree rooted at s (pred[s] = -1,    */
/* every walk reaches s in <= V-1 steps); (b) rebuild d along it, d[s] = 0,  */
/* d[v] = min over the arcs pred[v]->v of fl(d[pred[v]] + w) (a left-to-     */
/* right path sum, so d >= the BF fixpoint); (c) every arc satisfies         */
/* d[v] <= fl(d[u] + w) for finite d[u] (so d <= every path sum: d IS the    */
/* fixpoint, unreachable vertices included); (d) pred is canonical (O3) for  */
/* that d: the smallest steep tight tail; rows with a flat vertex or a       */
/* negative weight are compared whole with orc_pred on the rebuilt d.        */
/* Returns the number of rows failing; *first_bad = the first such row.      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int V; long long E; const int *src, *dst; const void *w; int wtype; int has_neg;
    const long long *in_ptr, *in_arc;
    const int *sources; int S; const int *pred; long long *bad; long long first_bad;
    int next; pthread_mutex_t mu;
} pcert_job;

static int pcert_row(pcert_job *j, int k, int *depth, int *stack, void *dv, int *canon)
{
    const int V = j->V, s = j->sources[k];
    const int *p = j->pred + (size_t)V * k;
    int *di = (int *)dv;
    float *df = (float *)dv;
    if (s < 0 || s >= V || p[s] != -1) return 1;
    for (int v = 0; v < V; ++v) {
        depth[v] = -1;
        if (j->wtype == ORC_I32) di[v] = I32_INF; else df[v] = INFINITY;
    }
    depth[s] = 0;
    if (j->wtype == ORC_I32) di[s] = 0; else df[s] = 0.0f;
    /* (a) + (b): walk up to a vertex with known d, then assign down */
    for (int v = 0; v < V; ++v) {
        if (depth[v] >= 0 || p[v] == -1) continue;
        int top = 0, x = v;
        while (depth[x] == -1) {
            if (p[x] < -1 || p[x] >= V) return 2;
            if (p[x] == -1) return 3;             /* a walk ending at a root != s */
            depth[x] = -2; stack[top++] = x; x = p[x];
        }
        if (depth[x] == -2) return 3;              /* cycle */
        while (top > 0) {
            int y = stack[--top], u = p[y], found = 0;
            depth[y] = depth[u] + 1;
            if (depth[y] > V - 1) return 3;
            for (long long q = j->in_ptr[y]; q < j->in_ptr[y + 1]; ++q) {
                long long e = j->in_arc[q];
                if (j->src[e] != u) continue;
                if (j->wtype == ORC_I32) {
                    int64_t c = (int64_t)di[u] + ((const int *)j->w)[e];
                    if (!found || c < di[y]) di[y] = (int)c;
                } else {
                    float c = df[u] + ((const float *)j->w)[e];
                    if (!found || c < df[y]) df[y] = c;
                }
                found = 1;
            }
            if (!found) return 4;                  /* pred[y] -> y is not an arc */
        }
    }
    /* (c) every arc */
    for (long long e = 0; e < j->E; ++e) {
        int u = j->src[e], v = j->dst[e];
        if (!finite_at(j->wtype, dv, u)) continue;
        if (j->wtype == ORC_I32) {
            if ((int64_t)di[u] + ((const int *)j->w)[e] < (int64_t)di[v]) return 5;
        } else {
            float c = df[u] + ((const float *)j->w)[e];
            if (c < df[v]) return 5;
        }
    }
    /* (d) canonical */
    int flat = j->has_neg;
    for (int v = 0; v < V && !flat; ++v) {
        if (v == s || p[v] < 0) continue;
        int best = -1;
        for (long long q = j->in_ptr[v]; q < j->in_ptr[v + 1]; ++q) {
            long long e = j->in_arc[q];
            int u = j->src[e];
            if (tight_arc(j->wtype, dv, j->w, e, u, v) && less_at(j->wtype, dv, u, v) && (best < 0 || u < best))
                best = u;
        }
        if (best < 0) flat = 1;
        else if (best != p[v]) return 6;
    }
    if (flat) {
        if (orc_pred(V, j->E, j->src, j->dst, j->w, j->wtype, s, dv, canon) != ORC_OK) return 7;
        if (memcmp(canon, p, sizeof(int) * (size_t)V) != 0) return 6;
    }
    return 0;
}

static void *pcert_worker(void *arg)
{
    pcert_job *j = (pcert_job *)arg;
    int *depth = (int *)malloc(sizeof(int) * (size_t)j->V);
    int *stack = (int *)malloc(sizeof(int) * (size_t)j->V);
    int *canon = (int *)malloc(sizeof(int) * (size_t)j->V);
    void *dv = malloc((size_t)4 * j->V);
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int k = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (k >= j->S) break;
        if (pcert_row(j, k, depth, stack, dv, canon)) {
            pthread_mutex_lock(&j->mu);
            *j->bad += 1;
            if (j->first_bad < 0 || k < j->first_bad) j->first_bad = k;
            pthread_mutex_unlock(&j->mu);
        }
    }
    free(depth); free(stack); free(canon); free(dv);
    return NULL;
}

long long orc_pred_certificate(int V, long long E, const int *src, const int *dst, const void *w,
                               int wtype, const int *sources, int S, const int *pred, int nthreads,
                               long long *first_bad)
{
    long long *in_ptr = (long long *)calloc((size_t)V + 1, sizeof(long long));
    long long *in_arc = (long long *)malloc(sizeof(long long) * (size_t)(E > 0 ? E : 1));
    long long *fill = (long long *)malloc(sizeof(long long) * (size_t)V);
    int has_neg = 0;
    if (wtype == ORC_I32)
        for (long long e = 0; e < E; ++e) if (((const int *)w)[e] < 0) has_neg = 1;
    for (long long e = 0; e < E; ++e) in_ptr[dst[e] + 1]++;
    for (int v = 0; v < V; ++v) in_ptr[v + 1] += in_ptr[v];
    memcpy(fill, in_ptr, sizeof(long long) * (size_t)V);
    for (long long e = 0; e < E; ++e) in_arc[fill[dst[e]]++] = e;
    long long bad = 0;
    pcert_job j = {V, E, src, dst, w, wtype, has_neg, in_ptr, in_arc, sources, S, pred, &bad, -1,
                   0, PTHREAD_MUTEX_INITIALIZER};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, pcert_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    if (first_bad) *first_bad = j.first_bad;
    free(in_ptr); free(in_arc); free(fill);
    return bad;
}
