"""Per-rank work of the sharded path, measured on ONE GPU (projection only).

For world W, runs every rank's phases (plan -> local BF + owned D entries ->
finish) one after another on cuda:0 with a loopback exchange (the rank-major
concatenation an all-gather produces) and reports each rank's device time.
The projected N-GPU step is max over ranks of (plan + local + finish) plus
the all-gather of W x max_send x 4 B at an assumed NVLink bandwidth; this is
a projection, NOT a multi-GPU measurement.

python tools/shard_probe.py --config 5 --worlds 1 2 4 8
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--nvlink-gbs", type=float, default=700.0, help="assumed all-gather bus bandwidth")
    ap.add_argument("--pred", action="store_true", help="also write each rank's pred rows (the bench's step)")
    a = ap.parse_args()
    import torch

    import gen
    import paper_2504_20655_b200 as wr
    torch.cuda.set_device(0)
    g, orders, _ = gen.config(a.config)
    G = wr.Graph.from_gen(g)
    dev = torch.device("cuda", 0)
    d_ptr = torch.from_numpy(orders.order_ptr).to(dev)
    d_nodes = torch.from_numpy(orders.order_nodes).to(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    warm = torch.empty((orders.B, wr.RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    for _ in range(2):   # warm the memory pool and the kernels
        wr.route_orders(G, d_ptr, d_nodes, results=warm)
    torch.cuda.synchronize()
    base = None
    pred_buf = [None]
    for W in a.worlds:
      for rep in range(2):   # the first pass of a world size warms allocations of its sizes
          per_rank = []
          plans = []
          for r in range(W):   # warm-up + plan timing
              e0, e1 = ev(), ev()
              e0.record()
              p = wr.OrdersPlan(G, d_ptr, d_nodes, r, W)
              if a.pred:
                  n_src = max(p.info.src_hi - p.info.src_lo, 1)
                  if pred_buf[0] is None or pred_buf[0].shape[0] < n_src:
                      pred_buf[0] = None
                      torch.cuda.empty_cache()
                      pred_buf[0] = torch.empty((n_src, g.V), dtype=torch.int32, device=dev)
                  p.close()
                  p = wr.OrdersPlan(G, d_ptr, d_nodes, r, W, pred_out=pred_buf[0])
              e1.record()
              torch.cuda.synchronize()
              plans.append((p, e0.elapsed_time(e1)))
          max_send = plans[0][0].info.max_send
          gathered = torch.zeros(W * max_send, dtype=torch.int32, device=dev)
          loc = []
          for r, (p, _) in enumerate(plans):
              st = p.local(gathered[r * max_send:(r + 1) * max_send])
              loc.append(st.ms)
          fin = []
          for r, (p, _) in enumerate(plans):
              n = p.info.order_hi - p.info.order_lo
              res = torch.empty((max(n, 1), wr.RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
              _, st = p.finish(gathered, results=res)
              fin.append(st.ms)
          for r in range(W):
              per_rank.append(plans[r][1] + loc[r] + fin[r])
          ag_ms = (W - 1) * max_send * 4 / (a.nvlink_gbs * 1e9) * 1e3 if W > 1 else 0.0
          step = max(per_rank) + ag_ms
          tput = orders.B / (step / 1e3)
          if rep == 0:
              for p, _ in plans:
                  p.close()
              continue
          base = base or tput
          print(json.dumps({"world": W, "projected_step_ms": step, "projected_orders_per_s": tput,
                            "projected_efficiency": tput / (base * W), "rank_ms_max": max(per_rank),
                            "rank_ms_min": min(per_rank), "plan_ms": max(p[1] for p in plans),
                            "local_ms_max": max(loc), "finish_ms_max": max(fin), "allgather_ms_assumed": ag_ms,
                            "max_send_bytes": max_send * 4, "pred": a.pred,
                            "measured_on": "1 GPU, ranks run sequentially"}),
                flush=True)
          for p, _ in plans:
              p.close()


if __name__ == "__main__":
    main()
