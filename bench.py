"""bench.py - routed orders/sec and edges relaxed/sec of the B200 hot path.

Workload (BASELINE.json configs[4], the metric's largest config that fits one
GPU): lattice(100,100,10) warehouse (V=100,000, E=968,040 arcs), 262,144
Zipf(1.0) orders of 6-8 picks -> ~84.7k distinct Bellman-Ford sources.
A step = one pass of the whole hot path over the batch: stop extraction
(a2), batched BF over every distinct stop (a3), canonical pred (a4), the D
gather (a5), exact routing of every order (a6), under the scheduler (a8);
at N>1 sources and orders are sharded and the owned D entries are
all-gathered over NCCL (a9). The graph is ingested (a1) once before timing.

Contract: python bench.py --gpus N --steps K --warmup W [--impl reference]
prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "edges relaxed/sec and routed orders/sec at 1/2/4/8 B200; HBM GB/s vs peak"
WORKLOAD = "configs[4]: 100k-location lattice(100,100,10), 968,040 arcs, 262,144 Zipf orders x 6-8 picks"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wr", choices=["wr", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--wtype", default="i32", choices=["i32", "f32"])
    ap.add_argument("--m", type=int, default=1, help="segments (1 = exact routes)")
    ap.add_argument("--pairs", action="store_true", help="segmented routes with the boundary-pair stitch (NEXT-1)")
    ap.add_argument("--nearfar", action="store_true", help="near-far deferral in the fp32 sweep (NEXT-3)")
    ap.add_argument("--depot", type=int, default=None, help="closed tours through this node (NEXT-4)")
    ap.add_argument("--no-pred", action="store_true", help="skip a4 (diagnostics only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(g, orders, seconds, S_total, m=1, pairs=False, depot=None):
    """The oracle as it stands, on the host cores, on a bounded sample: BF from
    a prefix of the distinct sources and exact routing of a prefix of the
    orders (their D rows recomputed by the oracle); extrapolated to the whole
    workload as B / (S * t_bf_per_source + B * t_route_per_order)."""
    import oracle
    threads = os.cpu_count() or 1
    stops_all = np.unique(orders.order_nodes)
    # sources: time one batch of `threads` sources, grow until ~seconds/2
    nsrc = min(threads, S_total)
    t_bf = None
    while True:
        t0 = time.perf_counter()
        oracle.bf_many(g, stops_all[:nsrc], nthreads=threads)
        dt = time.perf_counter() - t0
        t_bf = dt / nsrc
        if dt > seconds / 4 or nsrc >= min(4 * threads, S_total):
            break
        nsrc = min(nsrc * 2, S_total)
    # orders: route a prefix (the oracle BF for their stops is charged above)
    from gen.warehouse import Orders
    nord = min(64, orders.B)
    while True:
        sub = Orders(order_ptr=orders.order_ptr[:nord + 1].copy(),
                     order_nodes=orders.order_nodes[:int(orders.order_ptr[nord])].copy())
        sstops = np.unique(sub.order_nodes)
        t0 = time.perf_counter()
        res = oracle.route_orders(g, sub, m=m, nthreads=threads, pairs=pairs,
                                  depot=-1 if depot is None else depot)
        dt = time.perf_counter() - t0
        assert res["rc"] == 0
        t_route = max(0.0, (dt - t_bf * sstops.size)) / nord
        if dt > seconds / 2 or nord >= min(4096, orders.B):
            break
        nord = min(nord * 4, orders.B)
    B = orders.B
    t_full = S_total * t_bf + B * t_route
    return {"value": B / t_full, "unit": "orders/s", "cores": threads, "kind": "oracle",
            "sample": f"BF from {nsrc} of {S_total} distinct sources ({t_bf*1e3:.1f} ms/source on {threads} "
                      f"threads) + routing of the first {nord} orders ({t_route*1e3:.3f} ms/order); "
                      f"extrapolated to all {B} orders", "extrapolated": True}


def workload_config(a, g, orders, S):
    """The config dict both arms print (same keys and values)."""
    return {"workload": WORKLOAD if a.config == 5 else f"configs[{a.config-1}]", "orders": orders.B,
            "sources": S, "V": g.V, "E": g.E, "m": a.m, "pred": not a.no_pred,
            "stitch": "boundary pairs (NEXT-1)" if a.pairs else ("paper O7" if a.m >= 2 else "exact"),
            "tour": "open" if a.depot is None else f"closed through node {a.depot} (NEXT-4)",
            "sweep": "near-far (NEXT-3)" if a.nearfar else "frontier",
            "l2": ("working set (dist rows 4*V*S = %.1f GB) >> 126 MB L2; no flush needed" % (4 * g.V * S / 1e9))
            if 4 * g.V * S > 4 * 126e6 else
            ("working set (dist rows 4*V*S = %.3f GB) is L2-sized: steps run L2-warm "
             "(a parity-case line, not the headline workload)" % (4 * g.V * S / 1e9))}


def run_reference(a):
    """--impl reference: the CPU oracle on the same config/metric, bounded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gen
    g, orders, meta = gen.config(a.config, wtype=a.wtype)
    S = int(np.unique(orders.order_nodes).size)
    per_step = []
    cb = None
    for s in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(g, orders, max(2.0, a.cpu_seconds / max(1, a.steps)), S, m=a.m, pairs=a.pairs,
                          depot=a.depot)
        if s >= a.warmup:
            per_step.append(time.perf_counter() - t0)
    val = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "orders/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * orders.B / val,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": a.wtype,
            "data": "synthetic", "config": workload_config(a, g, orders, S),
            "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "orders/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s_per_sample": float(np.mean(per_step)) if per_step else None}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import gen
    import paper_2504_20655_b200 as wr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    g, orders, meta = gen.config(a.config, wtype=a.wtype)
    G = wr.Graph.from_gen(g, device=local)
    B = orders.B
    S = int(np.unique(orders.order_nodes).size)
    d_ptr = torch.from_numpy(orders.order_ptr).to(dev)
    d_nodes = torch.from_numpy(orders.order_nodes).to(dev)
    stream = torch.cuda.current_stream()

    rflags = (wr.WR_ROUTE_PAIRS if a.pairs else 0) | (wr.WR_ROUTE_NEARFAR if a.nearfar else 0)
    # N > 1: libwr's own context (NCCL communicator bootstrapped over the
    # process group): wr_route_orders shards sources and orders and runs the
    # all-gather of the owned D entries inside the call; each rank keeps its
    # own block of the results (WR_ROUTE_RANK_RESULTS)
    ctx = wr.Ctx.from_process_group(local) if world > 1 else None
    if world > 1:
        rflags |= wr.WR_ROUTE_RANK_RESULTS
    plan0 = wr.OrdersPlan(G, d_ptr, d_nodes, rank, world, m=a.m, stream=stream, flags=rflags)
    info = plan0.info
    n_my = info.order_hi - info.order_lo
    d_res = torch.empty((max(B, 1), wr.RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    pred_buf = None
    if not a.no_pred:
        pred_buf = torch.empty((max(int(info.src_hi - info.src_lo), 1), g.V), dtype=torch.int32, device=dev)
    plan0.close()
    launches = [0]
    bf_ms = [0.0]
    relax = [0]
    row_bits = [32]
    tiles = [0, 0]

    def step():
        _, st = wr.route_orders(G, d_ptr, d_nodes, m=a.m, results=d_res, stream=stream, pred_out=pred_buf,
                                flags=rflags, ctx=ctx, depot=a.depot)
        launches[0] += st.kernel_launches
        bf_ms[0] += st.bf_ms
        relax[0] += st.relaxations
        row_bits[0] = st.row_bits
        tiles[0], tiles[1] = st.tiles, st.tile_sources

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    launches[0] = 0
    bf_ms[0] = 0.0
    relax[0] = 0
    clocks = Clocks(local)
    barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    t = torch.tensor([ms, bf_ms[0] / a.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, bf_step_ms = float(t[0]), float(t[1])

    # e2e: the public C-ABI call with HOST buffers (pinned inputs copied in,
    # results copied out inside the call), N=1 path; sharded runs time the
    # phases with host inputs.
    e2e = None
    if not a.no_e2e:
        h_ptr = torch.from_numpy(orders.order_ptr).pin_memory()
        h_nodes = torch.from_numpy(orders.order_nodes).pin_memory()
        # results land in pinned host memory too (a pageable buffer would make
        # the device-to-host copy a staged, synchronous one)
        h_res_t = torch.empty(max(B, 1) * wr.RESULT_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
        h_res = h_res_t.numpy().view(wr.RESULT_DTYPE)

        def e2e_step():
            wr.route_orders(G, h_ptr.numpy(), h_nodes.numpy(), m=a.m, results=h_res, stream=stream, flags=rflags,
                            pred_out=pred_buf, ctx=ctx, depot=a.depot)

        for _ in range(2):
            e2e_step()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        k2 = max(1, a.steps)
        for _ in range(k2):
            e2e_step()
        f1.record(stream)
        barrier()
        ems = f0.elapsed_time(f1) / k2
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te[0])
        e2e = {"value": B / (ems / 1e3), "unit": "orders/s",
               "h2d_bytes_per_step": int(orders.order_ptr.nbytes + orders.order_nodes.nbytes),
               "d2h_bytes_per_step": int(n_my * wr.RESULT_DTYPE.itemsize) * world, "ms_per_step": ems}

    if ctx is not None:
        ctx.close()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm_peak, peak_kind = peaks()
    E = g.E
    useful = S * E                                    # graph500 convention: each arc once per source
    # roofline of the dominant kernel (the relaxation sweep): algorithmic bytes
    # per launch = compulsory traffic: write each
    # source's V distances once (4V per source, 2V with packed 16-bit rows)
    # + read the graph (in-arcs (u, w) 8E, out-arcs 4E, offsets 8V) once per
    # tile (128 sources, 256 packed).
    rb = row_bits[0] or 32
    # this rank's sources and the tiles its sweep actually ran (the tile
    # width follows choose_spl, narrower on shards)
    S_rank = int(info.src_hi - info.src_lo)
    alg_bytes = S_rank * (g.V * rb // 8) + tiles[0] * (12 * E + 8 * g.V)
    if not a.no_pred:
        # the canonical-pred pass (a4) runs fused inside the same kernel: it
        # reads every distance once more and writes every int32 pred once
        alg_bytes += S_rank * g.V * (rb // 8 + 4)
    bf_s = bf_step_ms / 1e3
    achieved = alg_bytes / bf_s / 1e9 if bf_s > 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    # DRAM bytes per launch from the committed ncu capture; that capture ran
    # the default workload (config 5, int32 weights, exact routes, fused pred),
    # so any other configuration reports null rather than someone else's bytes
    captured = (a.config == 5 and a.wtype == "i32" and a.m == 1 and not a.pairs and not a.no_pred
                and a.depot is None and not a.nearfar)
    if captured and os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("bf_frontier_kernel", {}).get("dram_bytes")
    # ALU view: one DPX add-min lane-op per useful relaxation (packed rows:
    # VIADDMNMX.U16x2, two relaxations per lane-op). Peak = the measured DPX
    # rate on this GPU model (tools/dpx_peak.cu: 1 warp instruction / clk /
    # SM for both forms -> profiles/r02_dpx_peak.jsonl), scaled to the clock
    # seen under load; fp32 rows add and min with two instructions, so the
    # 32-bit figure is an upper bound there
    clk = (ck.get("sm_mhz") or 1965.0) * 1e6
    dpx = {}
    dpath = os.path.join(ROOT, "profiles", "r02_dpx_peak.jsonl")
    if os.path.exists(dpath):
        for ln in open(dpath):
            r = json.loads(ln)
            dpx[r["op"]] = r["warp_instr_per_clk_per_sm"] * 32 * r["sms"]
    lanes = dpx.get("VIADDMNMX.U16x2" if rb == 16 else "VIADDMNMX.U32", 148 * 32)
    alu_peak = lanes * clk * (2 if rb == 16 else 1)
    alu_ach = useful / bf_s if bf_s > 0 else None
    line = {
        "metric": METRIC, "value": B / (ms / 1e3), "unit": "orders/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": a.wtype, "data": "synthetic",
        "config": workload_config(a, g, orders, S),
        "bf_rows": ("packed u16x2 keys (d << 4 | pred index), exact (bound checked, else packed / 32-bit redo); "
                    "outputs int32") if rb == 16 else "32-bit",
        "edges_relaxed_per_sec": {"useful": useful / (ms / 1e3), "useful_bf_only": useful / bf_s if bf_s else None,
                                  "performed_bf_only": (relax[0] / a.steps) / bf_s if bf_s else None,
                                  "unit": "edges/s", "convention": "useful = S*E (one traversal of every arc per source)"},
        "bf_ms_per_step": bf_step_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak if achieved else None,
                     "traffic": traffic / 1e9 if traffic else None, "traffic_unit": "GB per launch",
                     "algorithmic_gb_per_launch": alg_bytes / 1e9,
                     "kernel": "bf_frontier_kernel" + (" (a3 sweep + fused a4 pred pass)" if not a.no_pred else ""),
                     "peak_kind": peak_kind,
                     "note": "latency-bound frontier sweep; see DESIGN.md section 9"},
        "roofline_alu": {"bound": "alu", "achieved": alu_ach / 1e12 if alu_ach else None,
                         "peak": alu_peak / 1e12, "unit": "T relaxations/s",
                         "frac": alu_ach / alu_peak if alu_ach else None,
                         "peak_kind": "measured DPX rate (profiles/r02_dpx_peak.jsonl)" if dpx else "assumed"},
        "gpu_launches": int(launches[0]),
        "clocks": ck,
        "e2e": e2e,
    }
    if not a.no_cpu and world == 1:   # rank 0 at N=1 only
        line["cpu_baseline"] = cpu_baseline(g, orders, a.cpu_seconds, S, m=a.m, pairs=a.pairs, depot=a.depot)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
