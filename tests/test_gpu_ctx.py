"""The §8(b) boundary additions on the GPU: the library-owned NCCL context
(wr_ctx_create over a private one-rank communicator: the all-gather of the
owned D entries and the result exchange run inside libwr), wr_bf_batch's
stream-ordered async mode and shard option, and per-line caller labels on
wr_route_orders. Every result is compared with the CPU oracle. (World > 1
needs one GPU per rank - NCCL refuses two ranks on one device - so the
sharded phases themselves are covered by test_gpu_multiprocess.py with a
host-staged exchange, and by bench.py --gpus N.)"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2504_20655_b200 as wr  # noqa: E402


def _same(a, b):
    return a.tobytes() == b.tobytes()


@pytest.mark.parametrize("wtype,m,flags", [("i32", 1, 0), ("f32", 1, 0), ("i32", 3, wr.WR_ROUTE_PAIRS)])
def test_ctx_world1_route_orders_equals_plain_and_oracle(wtype, m, flags):
    cfg, B = (3, 2000) if m == 1 else (4, 300)
    g, orders, _ = gen.config(cfg, wtype=wtype, B=B)
    G = wr.Graph.from_gen(g)
    ctx = wr.Ctx(0, 1, None, 0)
    a, sa = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=m, flags=flags)
    b, sb = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=m, flags=flags, ctx=ctx)
    assert _same(a, b)
    c, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=m, flags=flags | wr.WR_ROUTE_RANK_RESULTS,
                           ctx=ctx)
    assert _same(a, c)
    exp = oracle.route_orders(g, orders, m=m, pairs=bool(flags & wr.WR_ROUTE_PAIRS))
    assert (exp["order_rc"] == 0).all()
    assert _same(wr.decode_cost(b, G.wtype), exp["cost"])
    assert np.array_equal(b["seq"], exp["seq"])
    # device results through the context as well
    d = torch.zeros((orders.B, wr.RESULT_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=m, flags=flags, ctx=ctx, results=d)
    assert d.cpu().numpy().tobytes() == a.tobytes()
    ctx.close()


def test_ctx_bf_batch_shard_world1_and_errors():
    g, orders, _ = gen.config(2)
    G = wr.Graph.from_gen(g)
    ctx = wr.Ctx(0, 1, None, 0)
    src = np.unique(orders.order_nodes)
    d0, p0, _ = wr.bf_batch(G, src, pred=True)
    d1, p1, _ = wr.bf_batch(G, src, pred=True, ctx=ctx, shard=True)
    assert _same(d0, d1) and _same(p0, p1)
    assert _same(d0, oracle.bf_many(g, src))
    with pytest.raises(wr.WrError) as e:
        wr.bf_batch(G, src, shard=True)
    assert e.value.code == wr.WR_EINVAL
    ctx.close()
    with pytest.raises(wr.WrError) as e:
        wr.Ctx(1, 1, None, 0)
    assert e.value.code == wr.WR_EINVAL
    with pytest.raises(wr.WrError) as e:
        wr.Ctx(0, 2, None, 0)   # world > 1 needs the unique id
    assert e.value.code == wr.WR_EINVAL
    assert len(wr.nccl_unique_id()) == wr.NCCL_UID_BYTES


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_bf_batch_async_returns_before_the_sweep_and_matches_oracle(wtype):
    """wr_bf_opts.async: the call returns with the sweep still running on
    the stream (an event recorded right after it is not yet complete);
    after a stream sync the rows equal the oracle."""
    g, orders, _ = gen.config(5, wtype=wtype, B=4000)
    G = wr.Graph.from_gen(g)
    src = np.unique(orders.order_nodes)[:2048].astype(np.int32)
    dist = torch.empty((src.size, g.V), dtype=torch.int32 if wtype == "i32" else torch.float32, device="cuda")
    pred = torch.empty((src.size, g.V), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    wr.bf_batch(G, src, pred=True, dist_out=dist, pred_out=pred, stream=s)   # warm (blocking)
    s.synchronize()
    dist.fill_(-5)
    pred.fill_(-5)
    _, _, st = wr.bf_batch(G, src, pred=True, dist_out=dist, pred_out=pred, stream=s, async_=True)
    ev = torch.cuda.Event()
    ev.record(s)
    pending = not ev.query()
    s.synchronize()
    assert pending, "the async call waited for its kernels"
    assert st.ms < 0
    rows = np.arange(0, src.size, 97)
    ref = oracle.bf_many(g, src[rows])
    assert _same(dist.cpu().numpy()[rows], ref)
    P = pred.cpu().numpy()
    assert np.array_equal(P[rows], oracle.pred_many(g, src[rows], ref))


@pytest.mark.parametrize("wtype,flags", [("i32", 0), ("f32", 0), ("i32", wr.WR_ROUTE_PAIRS)])
def test_route_orders_line_labels(wtype, flags):
    """Caller segment labels per order line (SURVEY §8(b) labels argument):
    every order is stitched over the caller's segments; equals the oracle's
    O7 / pair stitch on the oracle's own D with the same labels."""
    g, orders, _ = gen.config(4, wtype=wtype, B=120)
    rng = np.random.default_rng(17)
    node_label = rng.integers(0, 3, g.V).astype(np.int32)   # a label per node: lines at a node agree
    labels = node_label[orders.order_nodes]
    G = wr.Graph.from_gen(g)
    res, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes, labels=labels, flags=flags)
    for o in range(orders.B):
        nodes = orders.order_nodes[orders.order_ptr[o]:orders.order_ptr[o + 1]]
        stops = np.unique(nodes)
        D = oracle.bf_many(g, stops)[:, stops]
        fn = oracle.segmented_pairs_route if flags else oracle.segmented_route
        out = fn(D, node_label[stops])
        cost, seq = out[0], out[1]
        assert wr.decode_cost(res[o:o + 1], G.wtype)[0] == cost
        assert res["seq"][o][:stops.size].tolist() == stops[np.asarray(seq)].tolist()
    bad = labels.copy()
    o0 = int(np.argmax(np.diff(orders.order_ptr) > 0))
    bad[orders.order_ptr[o0]] = -1
    with pytest.raises(wr.WrError) as e:
        wr.route_orders(G, orders.order_ptr, orders.order_nodes, labels=bad)
    assert e.value.code == wr.WR_EINVAL
