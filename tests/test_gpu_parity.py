"""GPU parity: the CUDA path through the C-ABI against the CPU oracle, element
by element on the same seeded inputs. Bar (north star): dist and route cost
bit-exact for int32 AND fp32; pred equal to the canonical predecessor (O3);
route sequences equal (lexicographic tie rules O5/O7)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import gen  # noqa: E402
import oracle  # noqa: E402

wr = pytest.importorskip("paper_2504_20655_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.set_device(0)


class G:
    def __init__(self, V, src, dst, w, xy=None):
        self.V, self.src, self.dst, self.w = V, np.asarray(src, np.int32), np.asarray(dst, np.int32), np.asarray(w)
        self.xy, self.z = xy, None


def check_bf(g, sources, pred=True, variant=wr.WR_BF_AUTO, budget=0, targets=None):
    G = wr.Graph(g.V, g.src, g.dst, g.w, xy=getattr(g, "xy", None))
    dist, p, st = wr.bf_batch(G, sources, targets=targets, pred=pred and targets is None, variant=variant,
                              hbm_budget=budget)
    ref = oracle.bf_many(g, sources)
    if targets is not None:
        ref = ref[:, targets]
    assert dist.tobytes() == ref.tobytes()
    if pred and targets is None:
        for i, s in enumerate(sources):
            assert np.array_equal(p[i], oracle.pred(g, int(s), ref[i])), (i, s)
    return dist, p, st


# ------------------------------------------------------------------ a1
def test_graph_load_validation():
    with pytest.raises(wr.WrError) as e:
        wr.Graph(3, [0, 3], [1, 2], np.array([1, 1], np.int32))
    assert e.value.code == wr.WR_EINVAL
    for bad in (np.nan, -1.0, np.inf):
        with pytest.raises(wr.WrError) as e:
            wr.Graph(3, [0, 1], [1, 2], np.array([1.0, bad], np.float32))
        assert e.value.code == wr.WR_EINVAL
    with pytest.raises(wr.WrError) as e:
        wr.Graph(3, [0, 1], [1, 2], np.array([1, 2**30 + 5], np.int32))
    assert e.value.code == wr.WR_EOVERFLOW
    G = wr.Graph(4, [0, 1, 2], [1, 2, 3], np.array([1.0, -0.0, 2.0], np.float32))
    d, _, _ = wr.bf_batch(G, [0])
    assert d.tolist() == [[0.0, 1.0, 1.0, 3.0]] and not np.signbit(d).any()


def test_graph_csr_input_equals_coo():
    g = gen.config(2)[0]
    order = np.lexsort((g.dst, g.src))
    rp = np.zeros(g.V + 1, np.int64)
    np.add.at(rp, g.src[order] + 1, 1)
    rp = np.cumsum(rp)
    Gc = wr.Graph(g.V, row_ptr=rp, col=g.dst[order], w=g.w[order])
    Gd = wr.Graph(g.V, g.src, g.dst, g.w)
    srcs = np.arange(0, g.V, 7, dtype=np.int32)
    a, _, _ = wr.bf_batch(Gc, srcs)
    b, _, _ = wr.bf_batch(Gd, srcs)
    assert a.tobytes() == b.tobytes()


# ------------------------------------------------------------------ a3/a4
@pytest.mark.parametrize("wtype", ["i32", "f32"])
@pytest.mark.parametrize("k", [1, 2])
def test_bf_configs_all_sources(k, wtype):
    g = gen.config(k, wtype=wtype)[0]
    check_bf(g, np.arange(g.V, dtype=np.int32))


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_bf_config3_sample(wtype):
    g, orders, _ = gen.config(3, wtype=wtype, B=512)
    stops = np.unique(orders.order_nodes)
    check_bf(g, stops[:300])


@pytest.mark.parametrize("variant", [wr.WR_BF_FRONTIER, wr.WR_BF_DENSE])
def test_bf_variants_equal(variant):
    g = gen.config(2, wtype="f32")[0]
    check_bf(g, np.arange(0, g.V, 3, dtype=np.int32), variant=variant)


def test_bf_random_graphs_flat_and_absorption():
    """Zero weights, tiny weights (fp32 absorption) and multi-arcs exercise the
    flat-vertex path of the canonical pred."""
    rng = np.random.default_rng(5)
    for trial in range(30):
        V = int(rng.integers(2, 300))
        E = int(rng.integers(0, 5 * V))
        src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
        if trial % 2:
            w = rng.integers(0, 4, E).astype(np.int32)
        else:
            c = rng.integers(0, 4, E)
            w = np.select([c == 0, c == 1, c == 2], [np.zeros(E), np.full(E, 1e-8), 1e7 * rng.random(E)],
                          rng.random(E)).astype(np.float32)
        g = G(V, src, dst, w)
        check_bf(g, rng.integers(0, V, int(rng.integers(1, 70))).astype(np.int32))


def test_bf_negative_int_weights_and_negcycle():
    rng = np.random.default_rng(9)
    done = 0
    while done < 15:
        V = int(rng.integers(2, 60))
        E = int(rng.integers(V, 4 * V))
        g = G(V, rng.integers(0, V, E), rng.integers(0, V, E), rng.integers(-2, 8, E).astype(np.int32))
        srcs = rng.integers(0, V, 5).astype(np.int32)
        try:
            oracle.bf_many(g, srcs)
        except oracle.OracleError:
            with pytest.raises(wr.WrError) as e:
                wr.bf_batch(wr.Graph(g.V, g.src, g.dst, g.w), srcs)
            assert e.value.code == wr.WR_ENEGCYCLE
            continue
        check_bf(g, srcs)
        done += 1


def _neg_path(V=64, seed=11):
    """Bidirectional path 0 - 1 - ... - V-1: forward arcs 1..3 with one -1,
    backward arcs 5 (no negative cycle). From vertex 0 the shortest path to
    V-1 has V-1 hops, so Bellman-Ford still improves in round V-1 and must
    only stop after its check round V (§4.7, V-1 rounds)."""
    rng = np.random.default_rng(seed)
    fw = rng.integers(1, 4, V - 1).astype(np.int32)
    fw[V // 2] = -1
    src = list(range(V - 1)) + list(range(1, V))
    dst = list(range(1, V)) + list(range(V - 1))
    w = np.concatenate([fw, np.full(V - 1, 5, np.int32)])
    return G(V, src, dst, w, xy=np.stack([np.arange(V), np.zeros(V)], 1).astype(np.int32))


def test_bf_negative_weights_depth_v_minus_1():
    """Round-1 false WR_ENEGCYCLE: V = 2 with the single arc 0->1 (w = -1),
    and a 64-vertex path whose shortest path has V-1 hops; valid cycles
    still report WR_ENEGCYCLE. Through wr_bf_batch and wr_route_orders."""
    check_bf(G(2, [0], [1], np.array([-1], np.int32)), np.array([0, 1], np.int32))
    g = _neg_path()
    check_bf(g, np.array([0, 63, 31, 32], np.int32))
    Gp = wr.Graph(g.V, g.src, g.dst, g.w, xy=g.xy)
    _, _, st = wr.bf_batch(Gp, np.array([0], np.int32))
    assert st.rounds_max >= g.V - 1

    class O:
        pass
    orders = O()
    nodes = np.array([0, 63, 10, 40, 5, 63, 1, 62], np.int32)
    orders.order_ptr, orders.order_nodes, orders.B = np.array([0, 2, 5, 8], np.int64), nodes, 3
    compare_orders(g, orders, m=1, G=Gp)
    # the same path with a negative 2-cycle: 10 -> 11 (-1) -> 10 (-1)
    w2 = g.w.copy()
    w2[10] = -1
    w2[63 + 10] = -1
    Gc = wr.Graph(g.V, g.src, g.dst, w2, xy=g.xy)
    with pytest.raises(oracle.OracleError):
        oracle.bf_many(G(g.V, g.src, g.dst, w2, xy=g.xy), np.array([0], np.int32))
    for call in (lambda: wr.bf_batch(Gc, np.array([0, 5], np.int32)),
                 lambda: wr.route_orders(Gc, orders.order_ptr, orders.order_nodes)):
        with pytest.raises(wr.WrError) as e:
            call()
        assert e.value.code == wr.WR_ENEGCYCLE


def test_bf_flat_competing_predecessors():
    """The hand-derived O3 flat-rule fixtures of test_oracle_bf (competing
    tight tails with equal and different hop counts; steep beats flat) on
    the GPU: all sources, dist and pred equal to the oracle."""
    g = G(5, [0, 0, 1, 1, 2, 2, 3], [1, 2, 2, 3, 3, 4, 4], np.zeros(7, dtype=np.int32))
    check_bf(g, np.arange(5, dtype=np.int32))
    g2 = G(4, [0, 0, 2, 1, 2], [1, 2, 1, 3, 3], np.array([2, 1, 1, 0, 1], dtype=np.int32))
    check_bf(g2, np.arange(4, dtype=np.int32))
    g3 = G(5, [0, 0, 1, 1, 2, 2, 3], [1, 2, 2, 3, 3, 4, 4], np.zeros(7, dtype=np.float32))
    check_bf(g3, np.arange(5, dtype=np.int32))


def test_bf_long_path_many_rounds():
    """A 70,000-vertex path needs ~70k rounds from an end (more than 2^16):
    the sweep's round-stamped change words, word lists and the round-V
    negative-cycle test must still give the oracle's distances, preds and
    routes."""
    V = 70000
    a = np.arange(V - 1, dtype=np.int32)
    g = G(V, np.concatenate([a, a + 1]), np.concatenate([a + 1, a]), np.ones(2 * (V - 1), np.int32),
          xy=np.stack([np.arange(V), np.zeros(V)], 1).astype(np.int32))
    check_bf(g, np.array([0, 5, 40000], np.int32))
    Gp = wr.Graph(g.V, g.src, g.dst, g.w, xy=g.xy)

    class O:
        pass
    orders = O()
    nodes = np.array([0, 69999, 3, 65540, 32770, 7, 65536, 32768, 1], np.int32)
    orders.order_ptr, orders.order_nodes, orders.B = np.array([0, 2, 5, 9], np.int64), nodes, 3
    compare_orders(g, orders, m=1, G=Gp)


def test_bf_targets_repeats_and_device_outputs():
    g = gen.config(3, wtype="f32")[0]
    rng = np.random.default_rng(1)
    srcs = rng.integers(0, g.V, 77).astype(np.int32)
    srcs[5] = srcs[6]
    tg = rng.integers(0, g.V, 45).astype(np.int32)
    check_bf(g, srcs, targets=tg)
    G = wr.Graph.from_gen(g)
    d_dev = torch.empty((77, g.V), dtype=torch.float32, device="cuda")
    p_dev = torch.empty((77, g.V), dtype=torch.int32, device="cuda")
    wr.bf_batch(G, srcs, pred=True, dist_out=d_dev, pred_out=p_dev)
    d_host, p_host, _ = wr.bf_batch(G, srcs, pred=True)
    assert np.array_equal(d_dev.cpu().numpy(), d_host) and np.array_equal(p_dev.cpu().numpy(), p_host)


def test_bf_segment_budget_invariance():
    g = gen.config(3)[0]
    srcs = np.arange(0, g.V, 13, dtype=np.int32)   # 404 sources
    G = wr.Graph.from_gen(g)
    a, pa, sa = wr.bf_batch(G, srcs, pred=True)
    # rows + dist/pred staging = 12V bytes per source: room for 128-source
    # segments (one tile at the widest 32x4 layout)
    budget = G.info().device_bytes + (64 << 20) + 128 * 4 * g.V * 3 + 4096
    b, pb, sb = wr.bf_batch(G, srcs, pred=True, hbm_budget=budget)
    assert sa.segments == 1 and sb.segments > 1
    assert a.tobytes() == b.tobytes() and np.array_equal(pa, pb)


# ------------------------------------------------------------------ routes
def test_route_cost_vs_oracle():
    rng = np.random.default_rng(3)
    for dt in (np.int32, np.float32):
        n = 9
        D = (rng.random((n, n)) * 50).astype(dt)
        D[2, 5] = np.iinfo(np.int32).max if dt == np.int32 else np.inf
        seqs = np.array([rng.permutation(n) for _ in range(300)], dtype=np.int32)
        got = wr.route_cost(D, seqs)
        exp = np.array([oracle.route_cost(D, s) for s in seqs], dtype=dt)
        assert got.tobytes() == exp.tobytes()
    with pytest.raises(wr.WrError):
        wr.route_cost(np.zeros((3, 3), np.int32), np.array([[0, 3]], np.int32))


def test_route_segmented_worked_example():
    from test_oracle_bf import load_three_aisle
    rec = load_three_aisle()
    g = gen.aisle(3, 4, 2)
    G = wr.Graph.from_gen(g)
    r = wr.route_segmented(G, rec["picks"], m=1)
    picks = np.array(rec["picks"])
    cost, seq, rank = rec["exact"][0], rec["exact"][1], rec["exact"][2]
    assert int(r["cost_bits"]) == cost and r["rank"] == rank and r["seq"][:5].tolist() == picks[seq].tolist()
    for labels, c, s in rec["segmented"]:
        r = wr.route_segmented(G, rec["picks"], labels=labels, m=3)
        assert int(r["cost_bits"]) == c and r["seq"][:5].tolist() == picks[s].tolist()


def test_segment_plan_vs_oracle():
    rng = np.random.default_rng(17)
    for trial in range(200):
        n = int(rng.integers(1, 17))
        K = int(rng.integers(1, 5))
        span = int(rng.choice([3, 40, 1 << 19]))
        xy = rng.integers(-span, span, (n, 2)).astype(np.int32)
        assert wr.segment_plan(xy, K).tolist() == oracle.kmeans(xy, K).tolist(), (trial, n, K)


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_route_segmented_random_labels(wtype):
    g = gen.config(3, wtype=wtype)[0]
    G = wr.Graph.from_gen(g)
    rng = np.random.default_rng(23 if wtype == "i32" else 24)
    for trial in range(25):
        n = int(rng.integers(2, 13))
        stops = np.sort(rng.choice(5000, n, replace=False)).astype(np.int32)
        labels = rng.integers(0, min(6, n), n).astype(np.int32)
        r = wr.route_segmented(G, stops, labels=labels, m=6)
        D = oracle.bf_many(g, stops)[:, stops]
        c, s, counts = oracle.segmented_route(D, labels)
        assert wr.decode_cost(np.array([r]), G.wtype)[0].tobytes() == np.asarray(c).tobytes()
        assert r["seq"][:n].tolist() == stops[s].tolist()


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_route_segmented_pairs_random_labels(wtype):
    """NEXT-1 boundary-pair stitch through wr_route_segmented against the
    oracle's step-by-step definition (segments up to 9 stops)."""
    g = gen.config(3, wtype=wtype)[0]
    G = wr.Graph.from_gen(g)
    rng = np.random.default_rng(33 if wtype == "i32" else 34)
    for trial in range(25):
        n = int(rng.integers(2, 13))
        stops = np.sort(rng.choice(5000, n, replace=False)).astype(np.int32)
        labels = rng.integers(0, min(6, max(2, n // 3)), n).astype(np.int32)
        D = oracle.bf_many(g, stops)[:, stops]
        try:
            c, s, counts = oracle.segmented_pairs_route(D, labels)
        except oracle.OracleError as e:
            assert e.code == 6
            r = wr.route_segmented(G, stops, labels=labels, m=6, flags=wr.WR_ROUTE_PAIRS)
            assert r["status"] == wr.WR_ETOOLARGE
            continue
        r = wr.route_segmented(G, stops, labels=labels, m=6, flags=wr.WR_ROUTE_PAIRS)
        assert wr.decode_cost(np.array([r]), G.wtype)[0].tobytes() == np.asarray(c).tobytes()
        assert r["seq"][:n].tolist() == stops[s].tolist()


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_route_orders_pairs_config4(wtype):
    """C4 (10-11 stops, m = 3 O8 segments) with the boundary-pair stitch: every
    order equals the oracle; int costs never exceed the paper's stitch."""
    g, orders, _ = gen.config(4, wtype=wtype, B=256)
    G = wr.Graph.from_gen(g)
    res, st = compare_orders(g, orders, m=3, G=G, flags=wr.WR_ROUTE_PAIRS)
    assert st.stitch_candidates > 0
    if wtype == "i32":
        base, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=3)
        a, b = wr.decode_cost(res, G.wtype), wr.decode_cost(base, G.wtype)
        assert (a <= b).all() and (a < b).any()


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_route_orders_held_karp_13_to_16(wtype):
    """NEXT-2: exact routes of 13-16 stops (Held-Karp subset DP on the GPU)
    equal the oracle's (cost bits, order, rank); mixed with <= 12-stop orders
    routed by enumeration in the same call."""
    g = gen.config(3, wtype=wtype)[0]
    rng = np.random.default_rng(91 if wtype == "i32" else 92)
    sizes = [13, 14, 15, 16, 13, 16, 8, 12, 14, 5, 15, 16]
    nodes = np.concatenate([np.sort(rng.choice(5000, k, replace=False)) for k in sizes]).astype(np.int32)
    ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    class O:
        pass
    orders = O()
    orders.order_ptr, orders.order_nodes, orders.B = ptr, nodes, len(sizes)
    res, st = compare_orders(g, orders, m=1)
    assert res["n"].tolist() == sizes


def _absorption_graph(seed, near=24):
    """fp32 graph whose stop distances make rounding ties (reading A16): a
    complete digraph of `near` nodes with small weights (0.5 .. 3) and two
    far nodes joined to every near node by ~1e8 arcs (ulp 8), so every route
    through a far node absorbs the small prefix sums before its big leg."""
    rng = np.random.default_rng(seed)
    src, dst, w = [], [], []
    small = np.array([0.5, 1, 1.5, 2, 3], np.float32)
    for a in range(near):
        for b in range(near):
            if a != b:
                src.append(a); dst.append(b); w.append(rng.choice(small))
    for f in (near, near + 1):
        for a in range(near):
            src += [a, f]; dst += [f, a]
            w += [np.float32(1e8) + np.float32(8 * rng.integers(0, 4)), np.float32(1e8) + np.float32(8 * rng.integers(0, 4))]
    V = near + 2
    return G(V, src, dst, np.array(w, np.float32), xy=np.stack([np.arange(V), np.zeros(V)], 1).astype(np.int32))


def test_route_orders_held_karp_fp32_absorption():
    """NEXT-2 with fp32 absorption ties: 13-16-stop orders through the far
    nodes have many optimal orders whose prefixes differ in cost; the GPU
    (forward DP, backward bound, greedy) must return the oracle's O5 answer."""
    g = _absorption_graph(93)
    rng = np.random.default_rng(94)
    sizes = [13, 14, 15, 16] * 6
    seqs = []
    for k in sizes:
        far = rng.choice([24, 25], int(rng.integers(1, 3)), replace=False)
        near = rng.choice(24, k - far.size, replace=False)
        seqs.append(np.sort(np.concatenate([near, far])))
    nodes = np.concatenate(seqs).astype(np.int32)
    ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    class O:
        pass
    orders = O()
    orders.order_ptr, orders.order_nodes, orders.B = ptr, nodes, len(sizes)
    res, st = compare_orders(g, orders, m=1)
    assert (res["status"] == 0).all()


def _hk_digraph(seed, V=30, wmax=1000, neg=False, src_only=None, sink_only=None, ring=False):
    """Random digraph for the Held-Karp int paths: weights in [1, wmax), or
    reweighted by potentials (w + pi(u) - pi(v), some arcs negative, no
    negative cycle); optional out-arcs-only / in-arcs-only nodes (INF legs);
    ring: only arcs a -> a+1, a+3 (mod V), so legs span many arcs."""
    rng = np.random.default_rng(seed)
    pi = rng.integers(0, wmax // 2, V) if neg else np.zeros(V, np.int64)
    src, dst, w = [], [], []
    for a in range(V):
        for b in range(V):
            if ring:
                if (b - a) % V not in (1, 3):
                    continue
            elif a == b or rng.random() > 0.5 or a == sink_only or b == src_only:
                continue
            src.append(a); dst.append(b); w.append(int(rng.integers(wmax // 2 if ring else 1, wmax)) + int(pi[a]) - int(pi[b]))
    return G(V, src, dst, np.array(w, np.int32), xy=np.stack([np.arange(V), np.zeros(V)], 1).astype(np.int32))


@pytest.mark.parametrize("case", ["fast", "large_legs", "negative", "inf_legs"])
def test_route_orders_held_karp_int_paths(case):
    """NEXT-2 int32: the Held-Karp kernel's fast path (every leg finite and
    |leg| < 2^23: padded min/max, no INF tests) and its general path (a leg
    >= 2^23, or unreachable pairs) both equal the oracle (O5)."""
    kw = {"fast": dict(wmax=1000), "large_legs": dict(wmax=1 << 22, ring=True), "negative": dict(wmax=1000, neg=True),
          "inf_legs": dict(wmax=1000, src_only=3, sink_only=7)}[case]
    g = _hk_digraph(95, **kw)
    rng = np.random.default_rng(96)
    sizes = [13, 14, 15, 16, 8, 8] * 3   # 8 stops: the warp Held-Karp (same fast / general paths)
    seqs = []
    for k in sizes:
        pick = rng.choice(g.V, k, replace=False)
        if case == "inf_legs":
            pick = np.unique(np.concatenate([pick[: k - 2], [3, 7]]))
            while pick.size < k:
                pick = np.unique(np.concatenate([pick, rng.choice(g.V, 1)]))
        seqs.append(np.sort(pick))
    nodes = np.concatenate(seqs).astype(np.int32)
    ptr = np.concatenate([[0], np.cumsum([s.size for s in seqs])]).astype(np.int64)

    class O:
        pass
    orders = O()
    orders.order_ptr, orders.order_nodes, orders.B = ptr, nodes, len(seqs)
    res, _ = compare_orders(g, orders, m=1)
    assert (res["n"] >= 8).all()


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_route_orders_branch_and_bound_ties(wtype):
    """Exact enumeration with branch and bound (>= 9 stops, legs >= 0): on a
    graph where many or all routes tie (unit / zero weights) the strict bound
    test must keep O5's lexicographically smallest optimum; a random graph
    with a negative leg takes the unpruned path."""
    rng = np.random.default_rng(97)
    V = 24
    src, dst, w = [], [], []
    for a in range(V):
        for b in range(V):
            if a != b:
                src.append(a); dst.append(b)
                w.append(1 if (a + b) % 3 else (0 if wtype == "f32" else 2))
    dt = np.int32 if wtype == "i32" else np.float32
    g = G(V, src, dst, np.array(w, dt), xy=np.stack([np.arange(V), np.zeros(V)], 1).astype(np.int32))
    sizes = [9, 10, 9, 10, 9]
    seqs = [np.sort(rng.choice(V, k, replace=False)) for k in sizes]

    class O:
        pass
    orders = O()
    orders.order_ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    orders.order_nodes = np.concatenate(seqs).astype(np.int32)
    orders.B = len(sizes)
    compare_orders(g, orders, m=1)
    if wtype == "i32":   # one negative arc (no negative cycle): no pruning, same answers
        g2 = G(V, src, dst, np.array([x if i else -1 for i, x in enumerate(w)], np.int32), xy=g.xy)
        compare_orders(g2, orders, m=1)


def compare_orders(g, orders, m, chunk=0, G=None, results=None, flags=0):
    G = G or wr.Graph.from_gen(g)
    res, st = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=m, chunk=chunk, flags=flags) \
        if results is None else (results, None)
    exp = oracle.route_orders(g, orders, m=m, pairs=bool(flags & wr.WR_ROUTE_PAIRS))
    ok = exp["order_rc"] == 0
    assert np.array_equal(res["status"][ok], np.zeros(ok.sum()))
    cost = wr.decode_cost(res, G.wtype)
    assert cost[ok].tobytes() == exp["cost"][ok].tobytes()
    assert np.array_equal(res["seq"][ok], exp["seq"][ok])
    assert np.array_equal(res["rank"][ok], exp["rank"][ok])
    assert np.array_equal(res["n"], exp["n"])
    return res, st


@pytest.mark.parametrize("wtype", ["i32", "f32"])
@pytest.mark.parametrize("k,B", [(1, None), (2, None), (3, 1024)])
def test_route_orders_exact(k, B, wtype):
    g, orders, _ = gen.config(k, wtype=wtype, B=B)
    res, st = compare_orders(g, orders, m=1)
    # every order of <= 12 stops covers its n! sequences, however it is routed
    # (enumeration, branch and bound, or the 8-stop warp Held-Karp)
    ok = res["status"] == 0
    n = res["n"][ok]
    if n.size and n.max() <= 12:
        assert st.permutations == sum(math.factorial(int(x)) for x in n if x >= 2)


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_route_orders_segmented_config4(wtype):
    g, orders, _ = gen.config(4, wtype=wtype, B=256)
    res, st = compare_orders(g, orders, m=3)
    assert st.stitch_candidates > 0


def test_route_orders_exact_large_chunked():
    """C4 exact mode (n = 10-11, 14 chunks of <= 2,903,040 permutations) on a
    small sample; also a tiny chunk to force many work items."""
    g, orders, _ = gen.config(4, B=4)
    compare_orders(g, orders, m=1)
    g2, o2, _ = gen.config(2, B=32)
    compare_orders(g2, o2, m=1, chunk=50)


def test_route_orders_edge_cases():
    g = gen.config(2)[0]
    G = wr.Graph.from_gen(g)
    # empty order, single stop, duplicate lines, 17 distinct stops (too large)
    nodes = [5, 5, 5, 9, 7] + list(range(20, 37))
    ptr = np.array([0, 0, 3, 5, 5 + 17], np.int64)
    res, _ = wr.route_orders(G, ptr, np.array(nodes, np.int32))
    assert res["n"][:3].tolist() == [0, 1, 2]
    assert res["status"].tolist() == [0, 0, 0, wr.WR_ETOOLARGE]
    assert res["cost_bits"][1] == 0 and res["seq"][1][0] == 5
    assert sorted(res["seq"][2][:2].tolist()) == [7, 9] and res["seq"][3][0] == -1
    # unreachable stops: two components
    g2 = G_disconnected()
    G2 = wr.Graph(g2.V, g2.src, g2.dst, g2.w)
    res, _ = wr.route_orders(G2, np.array([0, 2, 4], np.int64), np.array([0, 1, 0, 3], np.int32))
    assert res["status"].tolist() == [0, wr.WR_EUNREACHABLE]


def test_frontier_size_limit_and_fallback_shape():
    """V beyond the shared-memory frontier -> WR_ETOOLARGE (documented in
    wr.h); V between the default and the fallback launch shape still routes
    exactly (path graph: dist = prefix sums)."""
    def path(V):
        src = np.arange(V - 1, dtype=np.int32)
        return wr.Graph(V, np.concatenate([src, src + 1]), np.concatenate([src + 1, src]),
                        np.ones(2 * (V - 1), np.int32))
    with pytest.raises(wr.WrError) as e:
        wr.bf_batch(path(250_000), [0], pred=False)
    assert e.value.code == wr.WR_ETOOLARGE
    G = path(150_000)
    d, p, _ = wr.bf_batch(G, [0, 149_999], pred=True)
    assert d[0].tolist() == list(range(150_000)) and d[1][0] == 149_999
    assert p[0][1:].tolist() == list(range(149_999)) and p[0][0] == -1


def G_disconnected():
    return G(4, [0, 1, 2, 3], [1, 0, 3, 2], np.array([1, 1, 1, 1], np.int32))


def test_route_orders_pred_rows():
    """a4 inside the orders path: pred rows of the distinct stops (ascending)
    equal the oracle's canonical predecessor; sharded ranks fill their own
    blocks and concatenate to the same matrix."""
    g, orders, _ = gen.config(3, wtype="f32", B=600)
    G = wr.Graph.from_gen(g)
    stops = np.unique(orders.order_nodes)
    pred = torch.full((stops.size, g.V), -7, dtype=torch.int32, device="cuda")
    wr.route_orders(G, orders.order_ptr, orders.order_nodes, pred_out=pred)
    P = pred.cpu().numpy()
    rows = oracle.bf_many(g, stops[::50])
    for k, i in enumerate(range(0, stops.size, 50)):
        assert np.array_equal(P[i], oracle.pred(g, int(stops[i]), rows[k]))
    world = 3
    parts = []
    for r in range(world):
        plan = wr.OrdersPlan(G, orders.order_ptr, orders.order_nodes, r, world)
        n = plan.info.src_hi - plan.info.src_lo
        pr = torch.full((max(n, 1), g.V), -7, dtype=torch.int32, device="cuda")
        plan = wr.OrdersPlan(G, orders.order_ptr, orders.order_nodes, r, world, pred_out=pr)
        send = torch.zeros(plan.info.max_send, dtype=torch.int32, device="cuda")
        plan.local(send)
        parts.append(pr.cpu().numpy()[:n])
    assert np.array_equal(np.concatenate(parts), P)


def _keyed_case(kind):
    """Graphs that select each row kind of the routing sweep with fused pred:
    keyed packed rows (small weights, in-degree <= 15), plain packed rows
    after a keyed overflow (a 300-vertex path of weight 100: distances to
    29,900 exceed the keyed 11-bit bound, fit 15 bits), plain packed rows
    for an in-degree-25 hub, 32-bit rows for weights > 0x3fff."""
    if kind == "keyed":
        return gen.config(3, B=400)[0]
    if kind == "path":
        V = 300
        src = list(range(V - 1)) + list(range(1, V))
        dst = list(range(1, V)) + list(range(V - 1))
        w = np.full(len(src), 100, np.int32)
        w[::7] = 37
        return G(V, src, dst, w, xy=np.stack([np.arange(V), np.zeros(V)], 1).astype(np.int32))
    if kind == "hub":
        n = 5
        src, dst, w = [], [], []
        for y in range(n):
            for x in range(n):
                v = y * n + x
                for dx, dy in ((1, 0), (0, 1)):
                    if x + dx < n and y + dy < n:
                        u = (y + dy) * n + x + dx
                        src += [v, u]; dst += [u, v]; w += [3, 3]
                src += [v, n * n]; dst += [n * n, v]; w += [2 + v % 5, 2 + v % 3]
        xy = np.array([(v % n, v // n) for v in range(n * n)] + [(9, 9)], np.int32)
        return G(n * n + 1, src, dst, np.array(w, np.int32), xy=xy)
    g = gen.config(3, B=400)[0]
    return G(g.V, g.src, g.dst, (g.w * 6000).astype(np.int32), xy=g.xy)


@pytest.mark.parametrize("kind,keyed,row_bits", [("keyed", 1, 16), ("path", 0, 16), ("hub", 0, 16),
                                                 ("wide", 0, 32)])
def test_route_orders_row_kinds_pred_and_routes(kind, keyed, row_bits):
    """Every row kind of the fused sweep (keyed / plain packed / 32-bit,
    including the keyed -> packed overflow redo) gives the oracle's routes
    and canonical pred rows (O3)."""
    g = _keyed_case(kind)
    rng = np.random.default_rng(71)
    B = 64
    n = rng.integers(3, 8, B)
    nodes = np.concatenate([rng.choice(g.V, k, replace=False) for k in n]).astype(np.int32)

    class O:
        pass
    orders = O()
    orders.order_ptr, orders.order_nodes, orders.B = np.concatenate([[0], np.cumsum(n)]).astype(np.int64), nodes, B
    Gd = wr.Graph(g.V, g.src, g.dst, g.w, xy=g.xy)
    stops = np.unique(nodes)
    pred = torch.full((stops.size, g.V), -7, dtype=torch.int32, device="cuda")
    res, st = wr.route_orders(Gd, orders.order_ptr, orders.order_nodes, pred_out=pred)
    assert (st.keyed, st.row_bits) == (keyed, row_bits)
    exp_rows = oracle.bf_many(g, stops)
    assert np.array_equal(pred.cpu().numpy(), oracle.pred_many(g, stops, exp_rows))
    compare_orders(g, orders, m=1, G=Gd, results=res)


def test_route_orders_budget_and_chunk_invariance():
    g, orders, _ = gen.config(3, B=2048)
    G = wr.Graph.from_gen(g)
    a, sa = wr.route_orders(G, orders.order_ptr, orders.order_nodes)
    budget = G.info().device_bytes + (128 << 20) + 256 * 4 * g.V
    b, sb = wr.route_orders(G, orders.order_ptr, orders.order_nodes, hbm_budget=budget, chunk=97)
    assert sb.segments > 1
    assert a.tobytes() == b.tobytes()


def _orders_with_pred(G, orders, S, V, flags=0):
    pred = torch.full((S, V), -7, dtype=torch.int32, device="cuda")
    res, st = wr.route_orders(G, orders.order_ptr, orders.order_nodes, pred_out=pred, flags=flags)
    return res, pred.cpu().numpy(), st


def test_packed_rows_equal_rows32():
    """Packed 16-bit working rows (int32 weights in [1, 0x3fff]) give the same
    routes, costs and pred rows as 32-bit rows (WR_ROUTE_ROWS32)."""
    g, orders, _ = gen.config(3, B=2048)
    assert int(np.min(g.w)) >= 1 and int(np.max(g.w)) <= 0x3fff   # the graph qualifies for packing
    G = wr.Graph.from_gen(g)
    S = np.unique(orders.order_nodes).size
    a, pa, _ = _orders_with_pred(G, orders, S, g.V)
    b, pb, _ = _orders_with_pred(G, orders, S, g.V, flags=wr.WR_ROUTE_ROWS32)
    assert a.tobytes() == b.tobytes()
    assert np.array_equal(pa, pb)
    compare_orders(g, orders, m=1, G=G, results=a)


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_fused_pred_segments_and_budget(wtype):
    """The pred pass fused into the sweep (CTAs out of tiles take pred jobs
    of finished tiles) gives the same rows with one segment and with many
    (small HBM budget), and the same rows as the standalone pred kernel of
    wr_bf_batch; spot rows equal the oracle's canonical pred."""
    g, orders, _ = gen.config(3, wtype=wtype, B=1024)
    G = wr.Graph.from_gen(g)
    stops = np.unique(orders.order_nodes)
    S = stops.size
    a, pa, sa = _orders_with_pred(G, orders, S, g.V)
    pred = torch.full((S, g.V), -7, dtype=torch.int32, device="cuda")
    budget = G.info().device_bytes + (128 << 20) + 256 * 4 * g.V
    b, sb = wr.route_orders(G, orders.order_ptr, orders.order_nodes, pred_out=pred, hbm_budget=budget)
    assert sb.segments > 1
    assert a.tobytes() == b.tobytes()
    assert np.array_equal(pa, pred.cpu().numpy())
    _, pb, _ = wr.bf_batch(G, stops[::37], pred=True)
    assert np.array_equal(pa[::37], pb)
    rows = oracle.bf_many(g, stops[::97])
    for k, i in enumerate(range(0, S, 97)):
        assert np.array_equal(pa[i], oracle.pred(g, int(stops[i]), rows[k]))


def _long_grid(n=24, w=0x3000):
    """n x n bidirectional grid with weights near the packed limit: distances
    reach ~2n*w >> 0x7fff, so a packed sweep must detect the overflow and
    redo the phase with 32-bit rows."""
    src, dst = [], []
    for i in range(n):
        for j in range(n):
            v = i * n + j
            if j + 1 < n:
                src += [v, v + 1]
                dst += [v + 1, v]
            if i + 1 < n:
                src += [v, v + n]
                dst += [v + n, v]
    rng = np.random.default_rng(7)
    ww = (w + rng.integers(0, 64, len(src))).astype(np.int32)
    xy = np.array([(v % n, v // n) for v in range(n * n)], np.int32)
    return G(n * n, src, dst, ww, xy=xy)


def test_packed_overflow_falls_back_exact():
    g = _long_grid()
    rng = np.random.default_rng(3)
    B = 64
    nodes = rng.integers(0, g.V, B * 5).astype(np.int32)
    ptr = np.arange(0, B * 5 + 1, 5, dtype=np.int64)

    class O:
        pass
    orders = O()
    orders.order_ptr, orders.order_nodes, orders.B = ptr, nodes, B
    G = wr.Graph(g.V, g.src, g.dst, g.w)
    S = np.unique(nodes).size
    res, P, _ = _orders_with_pred(G, orders, S, g.V)
    exp = oracle.route_orders(g, orders, m=1)
    assert wr.decode_cost(res, G.wtype).tobytes() == exp["cost"].tobytes()
    assert np.array_equal(res["seq"], exp["seq"])
    stops = np.unique(nodes)
    rows = oracle.bf_many(g, stops[::9])
    assert rows.max() > 0x7fff                       # the case really overflows 15 bits
    for k, i in enumerate(range(0, S, 9)):
        assert np.array_equal(P[i], oracle.pred(g, int(stops[i]), rows[k]))


# ------------------------------------------------------------------ a9
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_phases_equal_single(world):
    """Virtual ranks run one after another on one GPU; the all-gather is a
    rank-major concatenation of the padded send buffers (what
    torch.distributed.all_gather_into_tensor produces). No kernel waits on
    another rank."""
    g, orders, _ = gen.config(3, B=1500)
    G = wr.Graph.from_gen(g)
    ref, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes)
    plans = [wr.OrdersPlan(G, orders.order_ptr, orders.order_nodes, r, world) for r in range(world)]
    max_send = plans[0].info.max_send
    assert all(p.info.max_send == max_send for p in plans)
    gathered = torch.zeros(world * max_send, dtype=torch.int32, device="cuda")
    for r, p in enumerate(plans):
        p.local(gathered[r * max_send:(r + 1) * max_send])
    parts = [p.finish(gathered)[0] for p in plans]
    got = np.concatenate(parts)
    assert got.tobytes() == ref.tobytes()
    # and against the oracle directly (a9 parity, not only CUDA == CUDA)
    compare_orders(g, orders, m=1, G=G, results=got)


# ------------------------------------------------------------------ full size
@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_config5_full_size_sampled(wtype):
    """BASELINE.json configs[4] at full size (262,144 orders, 100k-vertex
    lattice, ~84.7k BF sources) in the bench's launch configuration; sampled
    orders and sources are recomputed by the oracle one by one."""
    g, orders, _ = gen.config(5, wtype=wtype)
    G = wr.Graph.from_gen(g)
    stops_all = np.unique(orders.order_nodes)
    pred_dev = torch.empty((stops_all.size, g.V), dtype=torch.int32, device="cuda")
    res, st = wr.route_orders(G, orders.order_ptr, orders.order_nodes, pred_out=pred_dev)
    assert st.sources == stops_all.size
    # pred rows of the bench's launch (packed rows for int32): sampled sources
    rng0 = np.random.default_rng(56)
    pick = np.sort(rng0.choice(stops_all.size, 6, replace=False))
    prow = pred_dev[torch.from_numpy(pick).cuda()].cpu().numpy()
    del pred_dev
    ref_rows = oracle.bf_many(g, stops_all[pick])
    for k, i in enumerate(pick):
        assert np.array_equal(prow[k], oracle.pred(g, int(stops_all[i]), ref_rows[k]))
    assert (res["status"] == 0).all()
    rng = np.random.default_rng(55)
    sample = np.sort(rng.choice(orders.B, 12, replace=False))
    for o in sample:
        nodes = orders.order_nodes[orders.order_ptr[o]:orders.order_ptr[o + 1]]
        stops = np.unique(nodes)
        rows = oracle.bf_many(g, stops)
        D = rows[:, stops]
        c, r, s = oracle.exact_route(D)
        assert wr.decode_cost(res[o:o + 1], G.wtype)[0] == c
        assert res["seq"][o][:stops.size].tolist() == stops[s].tolist() and res["rank"][o] == r
    # sampled full dist + pred rows of the same launch family
    srcs = np.sort(rng.choice(g.V, 40, replace=False)).astype(np.int32)
    dist, pred, _ = wr.bf_batch(G, srcs, pred=True)
    ref = oracle.bf_many(g, srcs)
    assert dist.tobytes() == ref.tobytes()
    for i in range(0, 40, 8):
        assert np.array_equal(pred[i], oracle.pred(g, int(srcs[i]), ref[i]))
    assert oracle.certificate(g, srcs, dist, pred) == 0
