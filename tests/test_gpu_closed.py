"""NEXT-4 closed tour through the depot (WR_ROUTE_CLOSED; reading R4: the
paper keeps entrance/exit out of the route, §3) on the GPU,
compared with the oracle's closed-tour functions on the same generated
warehouses: exact tours (enumerated, and Held-Karp for 13-16 stops), the
Theorem 3.1 stitch (O7) and the boundary-pair stitch, int32 and fp32,
orders with and without a line at the depot."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2504_20655_b200 as wr  # noqa: E402


class Orders:
    def __init__(self, lists):
        self.B = len(lists)
        self.order_ptr = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
        self.order_nodes = np.concatenate([np.asarray(x, np.int32) for x in lists]).astype(np.int32)


def depot_of(g):
    return g.V - 1 if g.name.startswith("aisle") else 0


def check(g, orders, m=1, flags=0, G=None):
    G = G or wr.Graph.from_gen(g)
    dep = depot_of(g)
    res, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=m, flags=flags, depot=dep)
    exp = oracle.route_orders(g, orders, m=m, pairs=bool(flags & wr.WR_ROUTE_PAIRS), depot=dep)
    ok = exp["order_rc"] == 0
    assert ok.all()
    assert (res["status"] == 0).all()
    assert np.array_equal(res["n"], exp["n"])
    assert wr.decode_cost(res, G.wtype).tobytes() == exp["cost"].tobytes()
    assert np.array_equal(res["seq"], exp["seq"])
    assert np.array_equal(res["rank"], exp["rank"])
    return res


@pytest.mark.parametrize("wtype", ["i32", "f32"])
@pytest.mark.parametrize("cfg,B", [(1, None), (2, None), (3, 1500)])
def test_closed_exact_configs(cfg, B, wtype):
    g, orders, _ = gen.config(cfg, wtype=wtype, B=B)
    res = check(g, orders)
    if cfg == 1:   # closing the tour never makes it cheaper than the open one
        G = wr.Graph.from_gen(g)
        op, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes)
        assert wr.decode_cost(res, G.wtype)[0] >= wr.decode_cost(op, G.wtype)[0]


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_closed_segmented_and_pairs_config4(wtype):
    g, orders, _ = gen.config(4, wtype=wtype, B=600)
    G = wr.Graph.from_gen(g)
    check(g, orders, m=3, G=G)
    check(g, orders, m=3, flags=wr.WR_ROUTE_PAIRS, G=G)
    # exact closed tours of 10-11 stops (11! in chunks) on a few orders
    lists = [orders.order_nodes[orders.order_ptr[o]:orders.order_ptr[o + 1]] for o in range(0, 600, 100)]
    check(g, Orders(lists), m=1, G=G)


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_closed_depot_as_a_stop_and_held_karp(wtype):
    """Orders with a line at the depot (it is then routed as a stop too),
    single-stop orders, and 13-15-stop orders (Held-Karp closed)."""
    g, _, _ = gen.config(3, wtype=wtype, B=10)
    dep = depot_of(g)
    rng = np.random.default_rng(88)
    lists = []
    for k in [1, 2, 3, 5, 7, 9]:
        nodes = list(rng.choice(g.V - 1, k, replace=False))
        lists.append(nodes + [dep])          # the depot is one of the stops
        lists.append(nodes)
    for k in [13, 14, 15, 15]:
        lists.append(list(rng.choice(g.V - 1, k, replace=False)))
    lists.append(list(rng.choice(g.V - 1, 14, replace=False)) + [dep, dep])   # 15 stops incl. the depot
    check(g, Orders(lists))


def test_closed_too_many_stops_and_bad_depot():
    g, _, _ = gen.config(3, B=10)
    G = wr.Graph.from_gen(g)
    rng = np.random.default_rng(89)
    o = Orders([list(rng.choice(g.V - 1, 16, replace=False)), [1, 2, 3]])
    res, _ = wr.route_orders(G, o.order_ptr, o.order_nodes, depot=g.V - 1)
    assert res["status"].tolist() == [wr.WR_ETOOLARGE, wr.WR_OK]   # 16 stops + the depot > 16
    with pytest.raises(wr.WrError) as e:
        wr.route_orders(G, o.order_ptr, o.order_nodes, depot=g.V)
    assert e.value.code == wr.WR_EINVAL


def test_closed_config5_sample():
    g, orders, _ = gen.config(5, B=2000)
    check(g, orders)
