"""Small end-to-end run for compute-sanitizer (configs 1-3, int and fp32,
exact + segmented routes, bf_batch with pred and targets)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gen  # noqa: E402
import paper_2504_20655_b200 as wr  # noqa: E402

for k, B in ((1, None), (2, 64), (3, 128), (4, 16)):
    for wt in ("i32", "f32"):
        g, orders, _ = gen.config(k, wtype=wt, B=B)
        G = wr.Graph.from_gen(g)
        stops = np.unique(orders.order_nodes)[:200]
        wr.bf_batch(G, stops, pred=True)
        wr.bf_batch(G, stops[:40], targets=stops[:17])
        wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=1)
        wr.route_orders(G, orders.order_ptr, orders.order_nodes, m=3)
        G.close()
print("sanitize run ok")
