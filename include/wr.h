/*
 * wr.h - C ABI of libwr, the B200-native hot path of arXiv:2504.20655
 * ("Warehouse storage and retrieval optimization via clustering, dynamical
 * systems modeling, and GPU-accelerated routing"): batched Bellman-Ford over
 * the warehouse picking graph, exhaustive route evaluation over pick-node
 * sequences, and the Theorem 3.1 segmented (cluster-stitched) route.
 *
 * Citations: P<line> = reference PAPER.md line (section); S<line> = SPEC.md
 * line; readings O1..O8 / A1..A19 are listed in DESIGN.md.
 *
 * Conventions (all functions):
 *  - extern "C", never throw or abort; return wr_status. WR_OK = 0.
 *  - wr_last_error() returns a thread-local message for the last failure.
 *  - Ownership: the caller owns every array passed in or out. Inputs are
 *    copied before the call returns; outputs are written only on WR_OK
 *    (contents unspecified on error). Opaque handles (wr_graph, wr_plan) are
 *    library-owned and released with the matching *_free.
 *  - Pointers may be host or device memory (detected with
 *    cudaPointerGetAttributes); device pointers must live on the graph's
 *    device. Host pointers may be pageable or pinned.
 *  - Calls are blocking by default. wr_bf_batch with opts.async = 1 and
 *    device outputs returns once its kernels are enqueued on opts.stream
 *    (results are stream-ordered; see wr_bf_opts.async for what it skips);
 *    the route calls are always blocking (their host-side plan needs the
 *    device's stop counts).
 *  - Every entry point opens an NVTX range named after it (nested ranges for
 *    the sweep, pred and route phases), visible to nsys / ncu --nvtx.
 *  - Sentinels: int32 INF = INT32_MAX, fp32 INF = +inf, pred NONE = -1,
 *    dist[s][s] = 0 (+0.0f).
 *  - Arithmetic: int32 sums are exact; fp32 sums are single IEEE-754
 *    binary32 round-to-nearest additions, left to right along a path or
 *    route (reading A6); no FMA, no flush-to-zero.
 */
#ifndef WR_H_
#define WR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t wr_status;
#define WR_OK 0
#define WR_EINVAL 1        /* bad argument, index, weight or size            */
#define WR_ENOMEM 2        /* device or host allocation failed               */
#define WR_ENEGCYCLE 3     /* a negative cycle is reachable (int weights)    */
#define WR_EOVERFLOW 4     /* int32 path/route sum bound exceeded (A7)       */
#define WR_EUNREACHABLE 5  /* stops of an order are not mutually reachable   */
#define WR_ETOOLARGE 6     /* problem exceeds a documented size limit        */
#define WR_ECUDA 7         /* CUDA runtime error                             */
#define WR_ENCCL 8         /* NCCL failure (wr_ctx communicator / collectives) */
#define WR_EINTERNAL 9

#define WR_I32 0           /* int32 weights / distances                      */
#define WR_F32 1           /* fp32 weights / distances                       */

#define WR_COO 0           /* arcs given as src[E], dst[E]                   */
#define WR_CSR 1           /* arcs given as out-adjacency row_ptr[V+1], col[E] */

#define WR_MAX_STOPS 16    /* stops per order (distinct location nodes)      */
#define WR_MAX_EXACT 12    /* stops of one exhaustively routed (sub)problem; */
                           /* exact orders of 13-16 stops use the Held-Karp  */
                           /* subset DP instead (same result, DESIGN R2)     */
#define WR_MAX_SEGMENTS 6  /* segments stitched per order (m'! 2^m' candidates) */
#define WR_DEFAULT_CHUNK 2903040LL /* permutations per chunk, P658 §4.6      */

const char *wr_last_error(void);
int32_t wr_version(void);
/* Device work memory comes from a per-device stream-ordered pool behind a
 * same-stream block cache: freed blocks are kept for the next call of the
 * same shape (no allocation driver call on repeated calls; an allocation
 * that fails releases the cache and retries). This returns every idle and
 * cached block to the driver (e.g. before handing the memory to another
 * allocator). */
wr_status wr_release_cached(int32_t device);

/* ------------------------------------------------ multi-GPU context (a9) -- */
/* One context per process and GPU, owning an NCCL
 * communicator over `world` ranks. Rank 0 calls wr_nccl_unique_id and the
 * caller broadcasts the 128 bytes to every rank (e.g. torch.distributed
 * broadcast_object_list); every rank then calls wr_ctx_create with its rank.
 * world = 1 may pass NULL (a private one-rank communicator). Calls that take
 * a context (wr_route_opts.ctx, wr_bf_opts.ctx + shard) are collective: all
 * ranks make the same call with the same inputs. NCCL is loaded at run time
 * (libnccl.so.2); failures map to WR_ENCCL. */
#define WR_NCCL_UID_BYTES 128
typedef struct wr_ctx wr_ctx;
wr_status wr_nccl_unique_id(void *uid_out);
wr_status wr_ctx_create(int32_t rank, int32_t world, const void *nccl_uid, int32_t device, wr_ctx **out);
wr_status wr_ctx_free(wr_ctx *ctx);
wr_status wr_ctx_info(const wr_ctx *ctx, int32_t *rank, int32_t *world, int32_t *device);

/* ---------------------------------------------------------------- graphs -- */
/* a1 Graph ingest (P721 §4.7: "edge-list format using integer arrays u, v,
 * and w"; S358-361 EdgeListGraph). Arcs are directed; an undirected edge is
 * two arcs. Multi-arcs allowed; self-loops allowed (never a predecessor).
 *   V        number of vertices, 1 <= V <= 2^30
 *   E        number of arcs, 0 <= E < 2^31
 *   wtype    WR_I32 or WR_F32
 *   format   WR_COO (src, dst used) or WR_CSR (row_ptr, col used)
 *   w        E weights of wtype, in arc order (COO order, or CSR order)
 *   xy       optional V x 2 int32 planar coordinates (|x|,|y| < 2^20) used
 *            by the default segment plan (O8) and to group nearby sources
 *            into Bellman-Ford tiles; NULL = none
 *   device   CUDA device ordinal
 *   z        optional V int32 rack level (|z| < 2^20), used with xy for the
 *            source tiling only; NULL = none
 * Validation: indices in [0, V); fp32 weights finite and >= 0 (-0.0 is
 * stored as +0.0); int32 weights any sign but (V-1) * max|w| < INT32_MAX
 * (else WR_EOVERFLOW). The device copy is a CSC (in-arcs sorted by (v,u))
 * plus CSR out-adjacency built by kernels on the device. */
typedef struct {
    int32_t V;
    int64_t E;
    int32_t wtype;
    int32_t format;
    const int32_t *src;
    const int32_t *dst;
    const int64_t *row_ptr;
    const int32_t *col;
    const void *w;
    const int32_t *xy;
    int32_t device;
    const int32_t *z;
} wr_graph_desc;

typedef struct wr_graph wr_graph;

typedef struct {
    int32_t V;
    int64_t E;
    int32_t wtype;
    int32_t has_negative;     /* any int weight < 0                          */
    int32_t has_xy;
    int32_t device;
    int64_t device_bytes;     /* bytes held on the device by the graph       */
    int32_t max_abs_weight;   /* int graphs: max |w|; fp32: 0                */
} wr_graph_info_t;

wr_status wr_graph_load(const wr_graph_desc *desc, wr_graph **out);
wr_status wr_graph_free(wr_graph *g);
wr_status wr_graph_info(const wr_graph *g, wr_graph_info_t *info);

/* ------------------------------------------------------- Bellman-Ford -- */
#define WR_BF_AUTO 0
#define WR_BF_FRONTIER 1   /* frontier-pull sweep over tiles of 32 sources   */
#define WR_BF_DENSE 2      /* every vertex every round (edge-parallel class) */
#define WR_BF_NEARFAR 3    /* NEXT-3 near-far deferral (fp32 graphs; int graphs
                              run WR_BF_FRONTIER): an improved vertex whose new
                              distances all exceed the tile's threshold T keeps
                              its row but propagates only once T reaches it; T
                              grows by delta = WR_NF_DELTA (default 0.75) x the
                              largest weight per round. Same results (O2
                              fixpoint); fewer relaxations, more rounds
                              (DESIGN §9 has the measured trade-off)        */

typedef struct {
    void *stream;            /* cudaStream_t; NULL = default stream          */
    int32_t async;           /* 1 with device dist/pred (or NULL), a graph
                                without negative weights and default
                                max_rounds: the call returns once the sweep
                                and output kernels are enqueued (no host sync
                                after the tiles are built); stats then hold
                                only segments/tiles/kernel_launches, ms = -1.
                                Otherwise ignored (blocking).               */
    int32_t variant;         /* WR_BF_*                                      */
    int32_t max_rounds;      /* relaxation rounds, 0 = V-1 (P724 §4.7); one
                                more round checks convergence: if it still
                                improves a distance -> WR_ENEGCYCLE (default
                                max_rounds, a negative cycle is reachable) or
                                WR_EINTERNAL (caller's max_rounds too small) */
    int64_t hbm_budget;      /* working-set bytes per segment; 0 = 180e9,
                                clamped to 90 % of free device memory (a8)  */
    wr_ctx *ctx;             /* optional multi-GPU context                  */
    int32_t shard;           /* 1 (needs ctx): rank r relaxes its contiguous
                                block of the S sources (wr_shard_range) and
                                the dist / pred row blocks are exchanged over
                                NCCL: every rank returns all S rows,
                                identical to an unsharded call              */
    int32_t reserved;        /* must be 0                                   */
} wr_bf_opts;

typedef struct {
    int32_t rounds_max;       /* most rounds any tile needed                 */
    int64_t relaxations;      /* (vertex, arc, source) relaxations performed */
    int32_t segments;         /* source batches the scheduler used           */
    int32_t tiles;            /* 32-source tiles                             */
    float ms;                 /* device time of the call (CUDA events)       */
    int32_t negcycle_source;  /* on WR_ENEGCYCLE: a source reaching one      */
    int64_t kernel_launches;  /* libwr kernels launched by the call          */
    int64_t visits;           /* (vertex, round) candidate visits, all tiles  */
} wr_bf_stats;

/* a3+a4 Batched Bellman-Ford (P720-724 §4.7: "dist and pred ... V x N,
 * where N denotes the number of source vertices processed simultaneously").
 *   sources  S source vertices (repeats allowed; rows follow input order)
 *   targets  T target vertices, or NULL for all V (then T is ignored, = V)
 *   dist     S x T row-major of the graph's wtype: dist[i][j] =
 *            shortest-path distance sources[i] -> targets[j], the unique
 *            fixpoint of d[v] = min(d[v], fl(d[u] + w)) (O2)
 *   pred     S x V int32 canonical predecessor (O3) or NULL
 *   stats    optional
 * Errors: WR_EINVAL (bad vertex), WR_ENEGCYCLE, WR_ENOMEM, WR_ECUDA,
 * WR_ETOOLARGE if V exceeds the shared-memory frontier (about 190,000
 * vertices on a B200: 36 bytes of per-vertex bitmaps, stamps and word lists
 * per CTA; the same limit applies to wr_route_orders). */
wr_status wr_bf_batch(const wr_graph *g, const int32_t *sources, int32_t S,
                      const int32_t *targets, int32_t T, void *dist, int32_t *pred,
                      const wr_bf_opts *opts, wr_bf_stats *stats);

/* --------------------------------------------------------------- routes -- */
/* O4 Route cost of caller-given sequences (P658 §4.6: "(n-1) transitions
 * must be evaluated to compute the total route cost"). Open route, depot
 * excluded (P322 §3).
 *   D      n x n row-major of wtype (directed, never mirrored, A15)
 *   seqs   count x len int32 indices into [0, n)
 *   costs  count results of wtype: cost = D[p0][p1] + ... left to right;
 *          len < 2 -> 0; any INF leg -> INF (not an error)
 * Errors: WR_EINVAL (index out of range, n < 1), WR_EOVERFLOW (int32). */
wr_status wr_route_cost(int32_t wtype, const void *D, int32_t n, const int32_t *seqs,
                        int32_t len, int64_t count, void *costs, void *stream);

typedef struct {
    void *stream;
    int32_t async;           /* reserved: route calls are blocking          */
    int32_t m;               /* 0/1: exact (O5); >= 2: segmented (O7) with  */
                             /* K = m O8 clusters when labels are not given */
    int64_t chunk;           /* permutations per chunk (O6); 0 = 2,903,040  */
    int64_t hbm_budget;      /* as in wr_bf_opts                            */
    int32_t *pred_out;       /* optional DEVICE int32 rows of V: canonical
                                pred (O3) of this call's BF sources, row =
                                index of the source in the ascending
                                distinct-stop list minus the rank's src_lo
                                (world 1: 0..S-1; rank r: its own block)    */
    int64_t pred_rows;       /* rows available in pred_out (>= src_hi-src_lo) */
    int32_t flags;           /* WR_ROUTE_* bits, 0 = defaults               */
    int32_t depot;           /* with WR_ROUTE_CLOSED: the depot node         */
    wr_ctx *ctx;             /* wr_route_orders only: NULL = this GPU alone;
                                a context shards the sources and orders over
                                its world (collective call, see below)      */
} wr_route_opts;

/* wr_route_opts.flags: keep the Bellman-Ford working rows in 32 bits even
 * when the graph admits packed 16-bit rows (int32 weights in [1, 0x3fff];
 * results are identical either way - a packed sweep whose distances could
 * exceed 0x7ffe is redone with 32-bit rows). */
#define WR_ROUTE_ROWS32 1
/* wr_route_opts.flags: segmented routing (m >= 2) with the boundary-pair
 * stitch (reading R1) instead of the paper's
 * fixed-route stitch (O7): per segment the best open path for every ordered
 * endpoint pair (first, last), then every segment order x one pair per
 * segment is costed left to right over the full sequence; min cost, ties ->
 * lexicographically smallest sequence. Segments <= 9 stops and
 * m'! * prod n_j (n_j - 1) <= 2^26 candidates, else WR_ETOOLARGE. */
#define WR_ROUTE_PAIRS 2
/* wr_route_opts.flags, with a context: write only this rank's block
 * [order_lo, order_hi) of the results (skips the result exchange). */
#define WR_ROUTE_RANK_RESULTS 4
/* wr_route_opts.flags: NEXT-4 closed tour (reading R4:
 * the paper leaves entrance/exit out of the route, P320 §3). Every order is
 * routed depot -> stops -> depot (opts.depot, a graph node), cost summed left
 * to right from the first depot leg; exact orders minimise the closed cost
 * over all orders of the stops (Held-Karp for 13-16), segmented ones keep the
 * segments' routes open and cost every stitch candidate as the closed tour.
 * The depot becomes a BF source; a closed order may hold at most 15 stops
 * other than the depot (WR_ETOOLARGE). Results list the order's own stops. */
#define WR_ROUTE_CLOSED 8
/* wr_route_opts.flags: run the routing path's sweep with WR_BF_NEARFAR. */
#define WR_ROUTE_NEARFAR 16

typedef struct {
    int32_t n;               /* stops (distinct nodes, ascending before routing) */
    int32_t status;          /* WR_OK, WR_EUNREACHABLE or WR_ETOOLARGE      */
    uint32_t cost_bits;      /* route cost, bit pattern of int32 or fp32    */
    int32_t m_used;          /* segments actually stitched (1 = exact)      */
    int64_t rank;            /* lexicographic rank of seq among n! orders   */
    int32_t seq[WR_MAX_STOPS]; /* node ids in visiting order, -1 padded     */
} wr_route_result;

typedef struct {
    int64_t orders;
    int64_t sources;          /* distinct stop nodes (BF sources)            */
    int64_t permutations;     /* sequences covered, segments + exact: enumerated, or proved no better (branch and bound, 8-stop Held-Karp); 13-16-stop Held-Karp orders add their DP transitions */
    int64_t stitch_candidates;
    int32_t segments;         /* BF source batches                           */
    int32_t rounds_max;
    int64_t relaxations;
    float ms;                 /* device time of the call                     */
    int64_t kernel_launches;
    float bf_ms;              /* device time of the relaxation sweeps alone  */
    float pred_ms;            /* device time of the canonical-pred pass      */
    int64_t visits;           /* BF candidate visits                         */
    int32_t row_bits;         /* BF working-row element width: 16 (packed,
                                 exact) or 32                                */
    int32_t keyed;            /* 1: the 16-bit rows carried (d << 4 | pred
                                 in-arc index) keys, so the fused pred pass
                                 only decoded them              */
    int64_t tiles;            /* BF source tiles swept (this rank)           */
    int32_t tile_sources;     /* sources per tile (row width)                */
    int32_t reserved2;
} wr_route_stats;

/* a7 Segmented route of one stop set (Theorem 3.1, P324-337 §3).
 *   stops   n node ids (deduplicated and sorted inside; n <= 16)
 *   labels  n segment labels aligned with the SORTED distinct stops, or NULL
 *           for the O8 plan (needs graph xy) with K = m
 *   m       segments (<= 1: exact route O5 over all n! sequences)
 * out: one wr_route_result. */
wr_status wr_route_segmented(const wr_graph *g, const int32_t *stops, int32_t n,
                             const int32_t *labels, int32_t m, const wr_route_opts *opts,
                             wr_route_result *out);

/* a2..a9 for a batch of orders (the production path, "routed orders/sec").
 *   order_ptr  B+1 int64 offsets into order_nodes
 *   order_nodes location node of each order line (P226-238 §2.4: lines at
 *              the same node are one stop)
 *   labels     optional segment label (>= 0) of each order line, aligned with
 *              order_nodes; lines at the same node must carry the same label
 *              (else WR_EINVAL). Given labels route every order by the stitch
 *              over the caller's segments (O7, or the pair stitch with
 *              WR_ROUTE_PAIRS; <= WR_MAX_SEGMENTS labels per order); NULL:
 *              opts.m decides (exact, or O8 K-means segments)
 *   results    B wr_route_result (host or device)
 * With opts.ctx (world W): rank r relaxes its block of the sorted distinct
 * stops, the owned D entries are all-gathered over NCCL on opts.stream, rank
 * r routes orders [order_lo, order_hi) (wr_shard_range) and the result
 * blocks are exchanged (grouped broadcasts) unless WR_ROUTE_RANK_RESULTS:
 * every rank's results equal the single-GPU call bit for bit. pred_out then
 * receives the rank's own source block (row 0 = its src_lo). stats are the
 * calling rank's. */
wr_status wr_route_orders(const wr_graph *g, const int64_t *order_ptr, const int32_t *order_nodes,
                          int64_t B, const int32_t *labels, const wr_route_opts *opts,
                          wr_route_result *results, wr_route_stats *stats);

/* O8 default segment plan for n points (labels in [0, min(m, n))). */
wr_status wr_segment_plan(const int32_t *xy, int32_t n, int32_t m, int32_t *labels_out,
                          int32_t device);

/* Theorem 3.1 counts (P326-329 §3; S430-438): reduced undirected count
 * m! 2^(m-1) + (1/2) sum n_j! and brute-force n!/2, n = sum n_j <= 20. */
wr_status wr_route_count_reduction(int32_t m, const int32_t *n_j, uint64_t *reduced,
                                   uint64_t *brute);

/* ------------------------------------------------ multi-GPU (a9) phases -- */
/* The sharded production path: every rank builds the same
 * plan; rank r runs Bellman-Ford for its contiguous block of the sorted
 * distinct sources and writes the D entries those sources own into a send
 * buffer; the caller all-gathers the send buffers (torch.distributed /
 * NCCL over NVLink, world x max_send elements); rank r then routes its
 * contiguous block of orders. Results equal wr_route_orders bit for bit
 * for any world size. */
typedef struct wr_plan wr_plan;

typedef struct {
    int64_t B;                /* orders in the batch                         */
    int64_t S;                /* distinct sources                            */
    int32_t rank, world;
    int64_t src_lo, src_hi;   /* this rank's source block                    */
    int64_t order_lo, order_hi; /* this rank's order block                   */
    int64_t send_count;       /* D entries this rank owns                    */
    int64_t max_send;         /* max over ranks (all-gather element count)   */
    int32_t wtype;
} wr_plan_info_t;

/* labels: as in wr_route_orders (per order line, or NULL). */
wr_status wr_orders_plan(const wr_graph *g, const int64_t *order_ptr, const int32_t *order_nodes,
                         int64_t B, const int32_t *labels, int32_t rank, int32_t world,
                         const wr_route_opts *opts, wr_plan **out);
wr_status wr_plan_info(const wr_plan *p, wr_plan_info_t *info);
/* send: device buffer of >= max_send 32-bit elements. */
wr_status wr_orders_local(wr_plan *p, void *send, const wr_route_opts *opts, wr_route_stats *stats);
/* gathered: device buffer, world x max_send elements (rank-major);
 * results: order_hi - order_lo entries (host or device). */
wr_status wr_orders_finish(wr_plan *p, const void *gathered, wr_route_result *results,
                           const wr_route_opts *opts, wr_route_stats *stats);
wr_status wr_plan_free(wr_plan *p);

/* Host-only helpers (no device needed), used by the CPU multi-rank tests. */
/* Contiguous block [lo, hi) of rank r when n units are split over world. */
void wr_shard_range(int64_t n, int32_t rank, int32_t world, int64_t *lo, int64_t *hi);

#ifdef __cplusplus
}
#endif
#endif /* WR_H_ */
