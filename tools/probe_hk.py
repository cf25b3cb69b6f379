"""NEXT-2 measurement: exact routes of 13-16-stop orders (Held-Karp on the
GPU) on the C3 warehouse; device time per call, orders/s, and the CPU
oracle's Held-Karp time per order on a small sample for context.

python tools/probe_hk.py [--B 1024] [--reps 3]
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
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--wtype", default="i32")
    a = ap.parse_args()
    import torch

    import gen
    import oracle
    import paper_2504_20655_b200 as wr
    torch.cuda.set_device(0)
    g = gen.config(3, wtype=a.wtype)[0]
    G = wr.Graph.from_gen(g)
    for n in (13, 14, 15, 16):
        rng = np.random.default_rng(1000 + n)
        nodes = np.concatenate([np.sort(rng.choice(5000, n, replace=False)) for _ in range(a.B)]).astype(np.int32)
        ptr = (np.arange(a.B + 1) * n).astype(np.int64)
        dptr = torch.from_numpy(ptr).cuda()
        dnodes = torch.from_numpy(nodes).cuda()
        res = torch.empty((a.B, wr.RESULT_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
        ms = []
        for r in range(a.reps + 1):
            _, st = wr.route_orders(G, dptr, dnodes, results=res)
            if r:
                ms.append(st.ms)
        # CPU oracle (Held-Karp in C, 1 thread per order) on 4 orders
        stops = nodes[:n]
        D = oracle.bf_many(g, stops)[:, stops]
        t0 = time.perf_counter()
        for _ in range(2):
            oracle.held_karp_route(D)
        t_cpu = (time.perf_counter() - t0) / 2
        print(json.dumps({"stops": n, "orders": a.B, "device_ms": float(np.median(ms)),
                          "orders_per_s": a.B / (np.median(ms) / 1e3), "dp_transitions_per_order": n * (n - 1) * 2 ** (n - 2),
                          "oracle_ms_per_order_1thread": t_cpu * 1e3}), flush=True)


if __name__ == "__main__":
    main()
