"""NEXT-3 near-far deferral (WR_BF_NEARFAR / WR_ROUTE_NEARFAR; PAPER.md:92
§1.1 names Δ-stepping as future work): the deferral only reorders the
chaotic relaxation, so dist is the same O2 fixpoint and pred the same
canonical O3 rows - compared element by element with the oracle on fp32
graphs with absorption and zero weights (flat vertices), on the aisle
configs and on a C5 sample, plus the routing path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2504_20655_b200 as wr  # noqa: E402
from test_gpu_parity import G, compare_orders  # noqa: E402


def _check(g, sources):
    Gd = wr.Graph(g.V, g.src, g.dst, g.w, xy=getattr(g, "xy", None))
    d, p, st = wr.bf_batch(Gd, sources, pred=True, variant=wr.WR_BF_NEARFAR)
    ref = oracle.bf_many(g, sources)
    assert d.tobytes() == ref.tobytes()
    assert np.array_equal(p, oracle.pred_many(g, sources, ref))
    return st


def test_nearfar_random_fp32_absorption_and_zero_weights():
    rng = np.random.default_rng(31)
    for trial in range(12):
        V = int(rng.integers(50, 400))
        E = int(rng.integers(V, 6 * V))
        src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
        k = rng.integers(0, 5, E)
        w = np.select([k == 0, k == 1, k == 2, k == 3],
                      [np.zeros(E), np.full(E, 1e-8), rng.uniform(0, 1, E), 1e6 * rng.uniform(0, 1, E)],
                      1e8 * rng.uniform(0, 1, E)).astype(np.float32)
        g = G(V, src, dst, w)
        _check(g, rng.choice(V, min(V, 70), replace=False).astype(np.int32))


@pytest.mark.parametrize("cfg", [2, 3])
def test_nearfar_aisle_configs(cfg):
    g, orders, _ = gen.config(cfg, wtype="f32", B=400)
    _check(g, np.unique(orders.order_nodes)[:300])


def test_nearfar_config5_sample_and_routes():
    g, orders, _ = gen.config(5, wtype="f32", B=1200)
    stops = np.unique(orders.order_nodes)
    st = _check(g, stops[::7][:256])
    assert st.relaxations > 0
    Gd = wr.Graph.from_gen(g)
    res, _ = wr.route_orders(Gd, orders.order_ptr, orders.order_nodes, flags=wr.WR_ROUTE_NEARFAR)
    compare_orders(g, orders, m=1, G=Gd, results=res)
    pred = torch.full((stops.size, g.V), -7, dtype=torch.int32, device="cuda")
    wr.route_orders(Gd, orders.order_ptr, orders.order_nodes, flags=wr.WR_ROUTE_NEARFAR, pred_out=pred)
    rows = np.arange(0, stops.size, 41)
    ref = oracle.bf_many(g, stops[rows])
    assert np.array_equal(pred.cpu().numpy()[rows], oracle.pred_many(g, stops[rows], ref))
