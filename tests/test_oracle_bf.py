"""Pins of the oracle's Bellman-Ford (O2) and canonical pred (O3) against
things other than itself: closed forms, an independent Dijkstra (heapq),
scipy's csgraph (library routine, int weights), Floyd-Warshall, the
hand-computed 3-aisle example, and the V1-V4 validity predicate.
CPU only."""
import heapq
import math
import os

import numpy as np
import pytest

import gen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


class G:  # minimal graph record accepted by the oracle front-end
    def __init__(self, V, src, dst, w):
        self.V = V
        self.src = np.asarray(src, dtype=np.int32)
        self.dst = np.asarray(dst, dtype=np.int32)
        self.w = np.asarray(w)


def unit_grid(nx, ny):
    """SPEC S376-384 build_grid_graph: unit 4-neighbour grid, both ways."""
    s, d = [], []
    for j in range(ny):
        for i in range(nx):
            v = j * nx + i
            if i + 1 < nx:
                s += [v, v + 1]; d += [v + 1, v]
            if j + 1 < ny:
                s += [v, v + nx]; d += [v + nx, v]
    return G(nx * ny, s, d, np.ones(len(s), dtype=np.int32))


def dijkstra(g, s):
    """Independent textbook Dijkstra with the same scalar arithmetic."""
    fp = g.w.dtype == np.float32
    adj = [[] for _ in range(g.V)]
    for u, v, w in zip(g.src.tolist(), g.dst.tolist(), g.w.tolist()):
        adj[u].append((v, np.float32(w) if fp else int(w)))
    inf = np.float32(np.inf) if fp else None
    d = [inf] * g.V
    d[s] = np.float32(0.0) if fp else 0
    pq = [(0.0, s)]
    done = [False] * g.V
    while pq:
        du, u = heapq.heappop(pq)
        if done[u]:
            continue
        done[u] = True
        for v, w in adj[u]:
            c = np.float32(d[u] + w) if fp else d[u] + w
            if d[v] is None or c < d[v]:
                d[v] = c
                heapq.heappush(pq, (float(c), v))
    if fp:
        return np.array(d, dtype=np.float32)
    return np.array([np.iinfo(np.int32).max if x is None else x for x in d], dtype=np.int32)


def random_graph(rng, V, E, kind):
    src = rng.integers(0, V, E)
    dst = rng.integers(0, V, E)
    if kind == "int":
        w = rng.integers(0, 21, E).astype(np.int32)
    else:
        choice = rng.integers(0, 5, E)
        w = np.select([choice == 0, choice == 1, choice == 2, choice == 3],
                      [np.zeros(E), np.full(E, 1e-8), rng.uniform(0, 1, E), 1e6 * rng.uniform(0, 1, E)],
                      1e8 * rng.uniform(0, 1, E)).astype(np.float32)
    return G(V, src, dst, w)


# ---------------------------------------------------------------- closed forms
def test_grid_arc_counts_spec_examples():
    assert unit_grid(2, 2).src.size == 8
    assert unit_grid(10, 10).src.size == 360
    assert unit_grid(1, 1).src.size == 0


def test_grid_manhattan():
    g = unit_grid(10, 10)
    d = oracle.bf(g, 0)
    assert d[99] == 18  # (1,1) -> (10,10), SPEC S392
    for s in (0, 37, 99):
        d = oracle.bf(g, s)
        sx, sy = s % 10, s // 10
        exp = [abs(v % 10 - sx) + abs(v // 10 - sy) for v in range(100)]
        assert d.tolist() == exp


def test_path_graph():
    g = G(3, [0, 1, 1, 2], [1, 0, 2, 1], np.ones(4, dtype=np.int32))
    assert oracle.bf(g, 0).tolist() == [0, 1, 2]


def aisle_formula(A, L, C, ws, wa, a, l, a2, l2):
    """closed-form slot distance on aisle(A, L, C)."""
    def y_slot(l):
        b = next(b for b in range(C - 1) if (b * L) // (C - 1) <= l < ((b + 1) * L) // (C - 1))
        return l + b + 1
    y1, y2 = y_slot(l), y_slot(l2)
    if a == a2:
        return ws * abs(y1 - y2)
    return min(ws * (abs(y1 - ((c * L) // (C - 1) + c)) + abs(y2 - ((c * L) // (C - 1) + c)))
               for c in range(C)) + wa * abs(a - a2)


@pytest.mark.parametrize("shape", [(3, 4, 2), (4, 10, 4), (10, 18, 2), (5, 9, 3), (7, 23, 5)])
@pytest.mark.parametrize("ws,wa", [(1, 3), (2, 5), (1, 1)])
def test_aisle_closed_form(shape, ws, wa):
    A, L, C = shape
    g = gen.aisle(A, L, C, ws=ws, wa=wa, wd=2)
    rng = np.random.default_rng(A * 100 + L)
    slots = A * L
    srcs = rng.choice(slots, size=min(slots, 6), replace=False)
    rows = oracle.bf_many(g, srcs)
    for s, row in zip(srcs, rows):
        a, l = divmod(int(s), L)
        for t in range(slots):
            a2, l2 = divmod(t, L)
            assert row[t] == aisle_formula(A, L, C, ws, wa, a, l, a2, l2), (s, t)


def test_generator_sizes():
    for dims, V, E in [((4, 10, 4), 57, 130), ((4, 10, 3), 53, 116), ((10, 18, 2), 201, 418),
                       ((50, 100, 5), 5251, 10892), ((3, 4, 2), 19, 40)]:
        g = gen.aisle(*dims)
        assert (g.V, g.E) == (V, E)
    g = gen.lattice(100, 100, 10)
    assert (g.V, g.E) == (100000, 968040)


# ------------------------------------------------------- the worked example
def load_three_aisle():
    rec = {"D": [], "segmented": [], "dist": [], "pred": []}
    for line in open(os.path.join(GOLD, "three_aisle.txt")):
        line = line.split("#")[0].split()
        if not line:
            continue
        k, rest = line[0], line[1:]
        if k == "picks":
            rec["picks"] = [int(x) for x in rest]
        elif k == "D":
            rec["D"].append([int(x) for x in rest])
        elif k == "exact":
            rec["exact"] = (int(rest[0]), [int(x) for x in rest[1].split(",")], int(rest[2]),
                            int(rest[3]), int(rest[4]))
        elif k == "segmented":
            rec["segmented"].append(([int(x) for x in rest[0].split(",")], int(rest[1]),
                                     [int(x) for x in rest[2].split(",")]))
        elif k == "closed":
            rec["closed"] = (int(rest[0]), [int(x) for x in rest[1].split(",")], int(rest[2]),
                             [int(x) for x in rest[3].split(",")], int(rest[4]), int(rest[5]))
        elif k in ("dist", "pred"):
            rec[k].append(tuple(int(x) for x in rest))
    rec["D"] = np.array(rec["D"], dtype=np.int32)
    return rec


def test_three_aisle_distances():
    rec = load_three_aisle()
    g = gen.aisle(3, 4, 2, ws=1, wa=3, wd=2)
    assert (g.V, g.E) == (19, 40)
    rows = oracle.bf_many(g, rec["picks"])
    D = rows[:, rec["picks"]]
    assert D.tolist() == rec["D"].tolist()
    for s, t, val in rec["dist"]:
        assert oracle.bf(g, s)[t] == val


def test_three_aisle_pred_tie():
    rec = load_three_aisle()
    g = gen.aisle(3, 4, 2, ws=1, wa=3, wd=2)
    for s, v, p in rec["pred"]:
        d = oracle.bf(g, s)
        assert oracle.pred(g, s, d)[v] == p


# ------------------------------------------------------------ Dijkstra pins
@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_bf_equals_dijkstra_random(kind):
    rng = np.random.default_rng(7 if kind == "int" else 8)
    for trial in range(150):
        V = int(rng.integers(2, 120))
        E = int(rng.integers(0, 4 * V))
        g = random_graph(rng, V, E, kind)
        s = int(rng.integers(0, V))
        got = oracle.bf(g, s)
        exp = dijkstra(g, s)
        assert got.tobytes() == exp.tobytes(), (trial, V, E)


def test_bf_equals_dijkstra_large_fp32_aisle():
    g = gen.aisle(10, 18, 2, wtype="f32", jitter_seed=5)
    for s in (0, 77, 200):
        assert oracle.bf(g, s).tobytes() == dijkstra(g, s).tobytes()


def test_bf_equals_scipy_int():
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra as sp_dijkstra
    rng = np.random.default_rng(11)
    for trial in range(40):
        V = int(rng.integers(2, 400))
        E = int(rng.integers(V, 6 * V))
        src = rng.integers(0, V, E)
        dst = rng.integers(0, V, E)
        w = rng.integers(1, 50, E).astype(np.int32)
        # scipy keeps the minimum of duplicate arcs only if we pre-reduce them
        key = src * V + dst
        order = np.lexsort((w, key))
        first = np.ones(E, dtype=bool)
        first[1:] = key[order][1:] != key[order][:-1]
        sel = order[first]
        M = csr_matrix((w[sel].astype(np.float64), (src[sel], dst[sel])), shape=(V, V))
        g = G(V, src, dst, w)
        for s in rng.integers(0, V, 3):
            exp = sp_dijkstra(M, indices=int(s))
            got = oracle.bf(g, int(s)).astype(np.float64)
            got[got == np.iinfo(np.int32).max] = np.inf
            assert np.array_equal(got, exp)


def test_bf_equals_floyd_warshall_with_negative_int():
    rng = np.random.default_rng(3)
    tested = 0
    while tested < 60:
        V = int(rng.integers(2, 24))
        E = int(rng.integers(V, 4 * V))
        src = rng.integers(0, V, E)
        dst = rng.integers(0, V, E)
        w = rng.integers(-3, 15, E).astype(np.int64)
        M = np.full((V, V), np.inf)
        np.fill_diagonal(M, 0)
        for u, v, x in zip(src, dst, w):
            M[u, v] = min(M[u, v], x)
        for k in range(V):
            M = np.minimum(M, M[:, k:k + 1] + M[k:k + 1, :])
        neg = np.any(np.diag(M) < 0)
        g = G(V, src, dst, w.astype(np.int32))
        for s in range(min(V, 4)):
            reach_neg = any(M[s, c] < np.inf and M[c, c] < 0 for c in range(V))
            if reach_neg:
                with pytest.raises(oracle.OracleError) as ei:
                    oracle.bf(g, s)
                assert ei.value.code == oracle.ENEGCYCLE
                continue
            got = oracle.bf(g, s).astype(np.float64)
            got[got == np.iinfo(np.int32).max] = np.inf
            assert np.array_equal(got, M[s]), (V, s)
            tested += 1
        del neg


def test_negative_cycle_fixture():
    # 0 -> 1 -> 2 -> 1 with cycle weight -1; 3 isolated with its own cycle
    g = G(5, [0, 1, 2, 3, 4], [1, 2, 1, 4, 3], np.array([1, 2, -3, -1, -1], dtype=np.int32))
    with pytest.raises(oracle.OracleError) as ei:
        oracle.bf(g, 0)
    assert ei.value.code == oracle.ENEGCYCLE
    # unreachable negative cycle does not matter
    g2 = G(5, [0, 3, 4], [1, 4, 3], np.array([4, -1, -1], dtype=np.int32))
    assert oracle.bf(g2, 0).tolist()[:2] == [0, 4]


# ---------------------------------------------------------- pred validity
def pred_valid(g, s, d, p):
    """Validity predicate V1-V4, written independently."""
    fp = g.w.dtype == np.float32
    inf = (lambda x: np.isinf(x)) if fp else (lambda x: x == np.iinfo(np.int32).max)
    V = g.V
    if p[s] != -1 or d[s] != 0:
        return "V1"
    arcs = {}
    for u, v, w in zip(g.src.tolist(), g.dst.tolist(), g.w.tolist()):
        arcs.setdefault((u, v), []).append(w)
    for v in range(V):
        if v == s:
            continue
        if inf(d[v]) != (p[v] == -1):
            return "V2"
        if p[v] == -1:
            continue
        u = int(p[v])
        ok = False
        for w in arcs.get((u, v), []):
            c = np.float32(d[u] + np.float32(w)) if fp else int(d[u]) + int(w)
            ok |= (not inf(d[u])) and c == d[v]
        if not ok:
            return "V3"
        x, steps = v, 0
        while x != s:
            x = int(p[x]); steps += 1
            if x < 0 or steps > V - 1:
                return "V4"
    return None


@pytest.mark.parametrize("kind", ["int", "fp32"])
def test_pred_valid_random(kind):
    rng = np.random.default_rng(21 if kind == "int" else 22)
    for trial in range(200):
        V = int(rng.integers(2, 60))
        E = int(rng.integers(0, 5 * V))
        g = random_graph(rng, V, E, kind)
        s = int(rng.integers(0, V))
        d = oracle.bf(g, s)
        p = oracle.pred(g, s, d)
        assert pred_valid(g, s, d, p) is None, trial


def test_pred_valid_negative_int():
    rng = np.random.default_rng(5)
    done = 0
    while done < 100:
        V = int(rng.integers(2, 30))
        E = int(rng.integers(0, 4 * V))
        g = G(V, rng.integers(0, V, E), rng.integers(0, V, E), rng.integers(-2, 6, E).astype(np.int32))
        s = int(rng.integers(0, V))
        try:
            d = oracle.bf(g, s)
        except oracle.OracleError:
            continue
        p = oracle.pred(g, s, d)
        assert pred_valid(g, s, d, p) is None
        done += 1


def test_pred_flat_zero_weight_cycle():
    # s=0 -> 1 (w 1); 1 <-> 2 (w 0); 2 -> 3 (w 0): flat vertices 2, 3
    g = G(4, [0, 1, 2, 2], [1, 2, 1, 3], np.array([1, 0, 0, 0], dtype=np.int32))
    d = oracle.bf(g, 0)
    assert d.tolist() == [0, 1, 1, 1]
    p = oracle.pred(g, 0, d)
    assert p.tolist() == [-1, 0, 1, 2]


def test_pred_flat_competing_predecessors_hand_derived():
    """O3's flat rule with competing tight predecessors, derived by hand.
    All-zero graph from s = 0: arcs 0->1, 0->2, 1->2, 1->3, 2->3, 2->4, 3->4.
    Every arc is tight and none is steep (d = 0 everywhere); hop over tight
    arcs: hop = [0, 1, 1, 2, 2]. pred[2]: tails 0 (hop 0), 1 (hop 1) -> 0;
    pred[3]: tails 1, 2 (both hop 1) -> the smaller, 1; pred[4]: tails 2
    (hop 1), 3 (hop 2) -> 2."""
    g = G(5, [0, 0, 1, 1, 2, 2, 3], [1, 2, 2, 3, 3, 4, 4], np.zeros(7, dtype=np.int32))
    d = oracle.bf(g, 0)
    assert d.tolist() == [0, 0, 0, 0, 0]
    assert oracle.pred(g, 0, d).tolist() == [-1, 0, 0, 1, 2]
    # mixed: 0->1 (2), 0->2 (1), 2->1 (1), 1->3 (0), 2->3 (1): d = [0, 2, 1, 2].
    # v = 1 has two steep tight tails (0, 2) -> the smaller, 0; v = 3 has a
    # flat tight tail 1 (d1 = d3) and a steep one 2 -> the steep rule wins, 2
    g2 = G(4, [0, 0, 2, 1, 2], [1, 2, 1, 3, 3], np.array([2, 1, 1, 0, 1], dtype=np.int32))
    d2 = oracle.bf(g2, 0)
    assert d2.tolist() == [0, 2, 1, 2]
    assert oracle.pred(g2, 0, d2).tolist() == [-1, 0, 0, 2]


def test_certificate_accepts_oracle_and_rejects_corruption():
    g = gen.aisle(4, 10, 4, wtype="f32", jitter_seed=9)
    srcs = np.array([0, 5, 17, 39, 56], dtype=np.int32)
    rows = oracle.bf_many(g, srcs)
    preds = np.stack([oracle.pred(g, s, r) for s, r in zip(srcs, rows)])
    assert oracle.certificate(g, srcs, rows, preds) == 0
    bad = rows.copy()
    bad[1, 20] = np.nextafter(bad[1, 20], np.float32(0))  # too small: no tight pred
    assert oracle.certificate(g, srcs, bad, preds) == 1
    bad = rows.copy()
    bad[2, 20] = np.nextafter(bad[2, 20], np.float32(np.inf))  # too big: arc violates
    assert oracle.certificate(g, srcs, bad, preds) == 1
    badp = preds.copy()
    badp[0, 3] = 3
    assert oracle.certificate(g, srcs, rows, badp) == 1


def test_paper_mteps_arithmetic():
    # P724 §4.7: 2627 MTEPS over E(V-1) edge visits at V=9716, E=26999
    visits = 26999 * (9716 - 1)
    assert visits == 262295285
    assert abs(visits / 2627e6 * 1e3 - 99.85) < 0.01
    assert math.ceil(26999 / 256) == 106


# ------------------------------------------- P9 from pred rows (full-size tier)
def _pc(g, srcs, P):
    return oracle.pred_certificate(g, srcs, P, nthreads=2)


def test_pred_certificate_accepts_oracle_rows():
    """Oracle pred rows (O3 on Dijkstra-pinned BF rows) pass: int and fp32
    aisle graphs, the worked example (pred ties), zero-weight flat vertices
    and negative int weights (both compared whole against orc_pred)."""
    cases = [gen.aisle(4, 10, 4, jitter_seed=3), gen.aisle(4, 10, 4, wtype="f32", jitter_seed=3),
             gen.aisle(3, 4, 2, ws=1, wa=3, wd=2),
             G(4, [0, 1, 2, 2], [1, 2, 1, 3], np.array([1, 0, 0, 0], dtype=np.int32)),
             G(5, [0, 1, 2, 0, 3], [1, 2, 3, 3, 4], np.array([4, -1, -2, 2, 1], dtype=np.int32))]
    for g in cases:
        srcs = np.arange(g.V, dtype=np.int32)
        rows = oracle.bf_many(g, srcs)
        P = oracle.pred_many(g, srcs, rows)
        for k in (0, g.V - 1):
            assert np.array_equal(P[k], oracle.pred(g, int(srcs[k]), rows[k]))
        assert _pc(g, srcs, P) == (0, -1)


def test_pred_certificate_rejects_corruption():
    """Each plausible GPU mistake fails the certificate: a non-canonical tie
    (the larger of two tight tails, worked example P3), a non-arc pred, a
    non-tight arc (a shortest-hop tree that is not a shortest-path tree), a
    2-cycle, a dropped reachable vertex, a pred on the source, and a row
    whose pred tree belongs to another source."""
    rec = load_three_aisle()
    g = gen.aisle(3, 4, 2, ws=1, wa=3, wd=2)
    srcs = np.arange(g.V, dtype=np.int32)
    rows = oracle.bf_many(g, srcs)
    P = oracle.pred_many(g, srcs, rows)
    # P3 tie: slot(0,2) -> slot(1,1) = 8 via the front and via the back cross
    # node: both tails are steep and tight, the canonical pred is the smaller
    s, v, p = next(t for t in rec["pred"] if t[0] == 2 and t[1] == 5)
    tails = [int(u) for u, x, w in zip(g.src, g.dst, g.w) if x == v and rows[s][u] + w == rows[s][v]]
    assert p == min(tails) and len(tails) >= 1
    mut = []
    bad = P.copy()
    other = [u for u in range(g.V) if u not in tails and u != v]
    alt = [t for t in rec["pred"] if t[0] == s]
    # non-canonical: any vertex with two steep tight tails
    for x in range(g.V):
        tt = sorted(int(u) for u, y, w in zip(g.src, g.dst, g.w)
                    if y == x and x != s and rows[s][u] + w == rows[s][x] and rows[s][u] < rows[s][x])
        if len(tt) >= 2:
            bad[s, x] = tt[1]
            mut.append(bad)
            break
    assert mut, alt
    nonarc = [u for u in other if not ((g.src == u) & (g.dst == v)).any()]
    bad = P.copy(); bad[s, v] = nonarc[0]; mut.append(bad)
    loose = [(int(u), int(x)) for u, x, w in zip(g.src, g.dst, g.w)
             if x != s and rows[s][u] + w > rows[s][x]]
    bad = P.copy(); bad[s, loose[0][1]] = loose[0][0]; mut.append(bad)   # real arc, not tight
    a, b = int(g.src[0]), int(g.dst[0])
    bad = P.copy(); bad[s, a] = b; bad[s, b] = a; mut.append(bad)    # 2-cycle (or wrong root)
    bad = P.copy(); bad[s, v] = -1; mut.append(bad)                  # reachable v dropped
    bad = P.copy(); bad[s, s] = int(P[s, v]); mut.append(bad)        # pred on the source
    bad = P.copy(); bad[s] = P[(s + 1) % g.V]; mut.append(bad)       # another source's tree
    for k, m in enumerate(mut):
        assert _pc(g, srcs, m) == (1, s), k
    # fp32: one ulp-wrong rebuilt sum cannot hide: a tree via a costlier tail
    gf = gen.aisle(4, 10, 4, wtype="f32", jitter_seed=9)
    sf = np.array([0, 17], dtype=np.int32)
    rf = oracle.bf_many(gf, sf)
    Pf = oracle.pred_many(gf, sf, rf)
    x = 20
    cand = [int(u) for u, y in zip(gf.src, gf.dst) if y == x and u != Pf[1, x]]
    ok = 0
    for u in cand:
        bad = Pf.copy(); bad[1, x] = u
        ok += _pc(gf, sf, bad) == (1, 1)
    assert ok == len(cand)
