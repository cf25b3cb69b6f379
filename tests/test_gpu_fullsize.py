"""Full-size verification tier (SURVEY.md §4 Tier 2, BASELINE.json configs):
the production launch (the bench's: packed rows, pred fused into the sweep)
checked against the CPU oracle at the configured sizes, not on samples.

* C5 (configs[4]), int32 (packed rows) and fp32 (32-bit rows): every one
  of the ~84.7k pred rows of the launch passes the oracle's P9 certificate
  from pred alone (a tree rooted at its source whose path sums satisfy every
  arc, i.e. ARE the BF fixpoint, with the canonical O3 tails), streamed in
  blocks through all host cores; every 16th row also equals the oracle's
  O3 pred of the oracle's own BF row (O2); 16,384 (int32) / 4,096 (fp32)
  of the 262,144 routed orders equal oracle.route_orders.
* C3 (configs[2]) at its full 16,384 orders, clustered and unclustered
  layouts, int32 and fp32.
* C4 (configs[3]) at its full 4,096 orders: the paper's stitch (O7, m = 3)
  and the boundary-pair stitch (NEXT-1); exact mode (m = 1, 11! in chunks)
  on 32 of them.

This is the paper's own validation idea (CPU BF = GPU BF, PAPER.md:730
Remark) at full size. Oracle inputs come only from gen/ and oracle/.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2504_20655_b200 as wr  # noqa: E402


class _Sub:
    """A subset of an Orders batch (the same orders, same line order)."""

    def __init__(self, orders, idx):
        idx = np.asarray(idx, np.int64)
        lens = orders.order_ptr[idx + 1] - orders.order_ptr[idx]
        self.order_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.order_nodes = np.concatenate(
            [orders.order_nodes[orders.order_ptr[o]:orders.order_ptr[o + 1]] for o in idx]).astype(np.int32)
        self.B = idx.size


def _check_results(res, wtype, exp, idx=None):
    sel = slice(None) if idx is None else idx
    r = res[sel]
    assert (exp["order_rc"] == 0).all()
    assert (r["status"] == 0).all()
    cost = wr.decode_cost(r, wtype)
    assert cost.tobytes() == exp["cost"].tobytes()
    assert np.array_equal(r["n"], exp["n"])
    assert np.array_equal(r["seq"], exp["seq"])
    assert np.array_equal(r["rank"], exp["rank"])


def _pred_rows_vs_oracle(g, stops, pred_dev, block=2048, every=16):
    """Every row of pred_dev (device, S x V) passes oracle.pred_certificate;
    every `every`-th row also equals O3 of the oracle's own BF row."""
    for b in range(0, stops.size, block):
        got = pred_dev[b:b + block].cpu().numpy()
        bad, first = oracle.pred_certificate(g, stops[b:b + block], got)
        assert bad == 0, f"{bad} pred rows fail the certificate, first at source {stops[b + first]}"
        ii = np.arange(b, min(b + block, stops.size))[::every]
        ref = oracle.bf_many(g, stops[ii])
        exp = oracle.pred_many(g, stops[ii], ref)
        diff = np.nonzero((got[ii - b] != exp).any(axis=1))[0]
        assert diff.size == 0, f"pred rows differ from the oracle at sources {stops[ii[diff[:8]]]}"


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_config5_production_launch_vs_oracle(wtype):
    g, orders, _ = gen.config(5, wtype=wtype)
    G = wr.Graph.from_gen(g)
    stops = np.unique(orders.order_nodes)
    pred_dev = torch.full((stops.size, g.V), -7, dtype=torch.int32, device="cuda")
    res, st = wr.route_orders(G, orders.order_ptr, orders.order_nodes, pred_out=pred_dev)
    assert st.sources == stops.size
    if wtype == "i32":
        assert st.row_bits == 16   # the bench's launch: packed u16 rows, fused pred
    _pred_rows_vs_oracle(g, stops, pred_dev)
    del pred_dev
    torch.cuda.empty_cache()
    rng = np.random.default_rng(5005)
    idx = np.sort(rng.choice(orders.B, 16384 if wtype == "i32" else 4096, replace=False))
    exp = oracle.route_orders(g, _Sub(orders, idx), m=1)
    _check_results(res, G.wtype, exp, idx)
    G.close()


@pytest.mark.parametrize("clustered", [False, True])
@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_config3_full_batch_both_layouts(wtype, clustered):
    g, orders, meta = gen.config(3, wtype=wtype, clustered=clustered)
    assert orders.B == 16384 and meta["clustered"] == clustered
    G = wr.Graph.from_gen(g)
    res, st = wr.route_orders(G, orders.order_ptr, orders.order_nodes)
    exp = oracle.route_orders(g, orders, m=1)
    _check_results(res, G.wtype, exp)
    G.close()


@pytest.mark.parametrize("wtype", ["i32", "f32"])
def test_config4_full_batch_stitches(wtype):
    g, orders, meta = gen.config(4, wtype=wtype)
    assert orders.B == 4096 and meta["m"] == 3
    G = wr.Graph.from_gen(g)
    for flags, pairs in ((0, False), (wr.WR_ROUTE_PAIRS, True)):
        res, _ = wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=3, flags=flags)
        exp = oracle.route_orders(g, orders, m=3, pairs=pairs)
        _check_results(res, G.wtype, exp)
    # exact mode (11! per order in 2,903,040-permutation chunks) on 32 orders
    sub = _Sub(orders, np.arange(0, 4096, 128))
    res, _ = wr.route_orders(G, sub.order_ptr, sub.order_nodes, m=1)
    exp = oracle.route_orders(g, sub, m=1)
    _check_results(res, G.wtype, exp)
    G.close()
