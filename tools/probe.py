"""Quick per-phase probe of the hot path on one GPU (diagnostics, not the bench).

python tools/probe.py --config 5 --reps 2 [--wtype f32] [--variant 1|2] [--bf-only]
Prints one JSON line per rep with BF / pred / routing device times and the
work counters libwr reports.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--wtype", default="i32")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--B", type=int, default=None)
    ap.add_argument("--pred", action="store_true")
    ap.add_argument("--bf-sources", type=int, default=0, help="run wr_bf_batch on the first N stops")
    a = ap.parse_args()
    import torch

    import gen
    import paper_2504_20655_b200 as wr
    torch.cuda.set_device(0)
    t0 = time.time()
    g, orders, meta = gen.config(a.config, wtype=a.wtype, B=a.B)
    G = wr.Graph.from_gen(g)
    dev = torch.device("cuda", 0)
    d_ptr = torch.from_numpy(orders.order_ptr).to(dev)
    d_nodes = torch.from_numpy(orders.order_nodes).to(dev)
    S = int(np.unique(orders.order_nodes).size)
    res = torch.empty((orders.B, wr.RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    pred = torch.empty((S, g.V), dtype=torch.int32, device=dev) if a.pred else None
    print(json.dumps({"setup_s": time.time() - t0, "V": g.V, "E": g.E, "S": S, "B": orders.B}), flush=True)
    for r in range(a.reps):
        torch.cuda.synchronize()
        t = time.time()
        _, st = wr.route_orders(G, d_ptr, d_nodes, m=a.m, results=res, pred_out=pred)
        torch.cuda.synchronize()
        wall = time.time() - t
        print(json.dumps({"rep": r, "wall_ms": wall * 1e3, "call_ms": st.ms, "bf_ms": st.bf_ms, "pred_ms": st.pred_ms,
                          "relaxations": st.relaxations, "visits": st.visits, "useful": S * g.E,
                          "work_ratio": st.relaxations / max(1, S * g.E), "rounds_max": st.rounds_max,
                          "permutations": st.permutations, "stitch": st.stitch_candidates,
                          "launches": st.kernel_launches,
                          "useful_gteps_bf": S * g.E / (st.bf_ms * 1e6) if st.bf_ms else None}), flush=True)
    if a.bf_sources:
        stops = np.unique(orders.order_nodes)[: a.bf_sources]
        out = torch.empty((stops.size, g.V), dtype=torch.int32 if a.wtype == "i32" else torch.float32, device=dev)
        for variant in (1, 2):
            torch.cuda.synchronize()
            _, _, st = wr.bf_batch(G, stops, dist_out=out, variant=variant)
            print(json.dumps({"bf_batch_variant": variant, "sources": int(stops.size), "ms": st.ms,
                              "rounds_max": st.rounds_max, "relaxations": st.relaxations,
                              "work_ratio": st.relaxations / (stops.size * g.E)}), flush=True)


if __name__ == "__main__":
    main()
