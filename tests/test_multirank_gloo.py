"""The N>1 path's host logic on CPU with torch.distributed (gloo, world 2):
sources sharded with libwr's wr_shard_range, each rank fills the send buffer
in the exchange layout libwr documents (wr.h "multi-GPU (a9) phases": orders
ascending, owned stops ascending, targets ascending; offsets = exclusive
scan of owned-row counts), one all_gather_into_tensor, each rank reassembles
D for its order block and routes it. The compute here is the CPU oracle
(test infrastructure); the GPU kernels of the same protocol are covered by
tests/test_gpu_parity.py::test_sharded_phases_equal_single."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rank_main(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import gen
    import oracle
    import paper_2504_20655_b200 as wr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, orders, _ = gen.config(2, B=96)
    B = orders.B
    stops = [np.unique(orders.order_nodes[orders.order_ptr[o]:orders.order_ptr[o + 1]]) for o in range(B)]
    sources = np.unique(orders.order_nodes)
    S = sources.size
    row = {int(v): i for i, v in enumerate(sources)}
    blk = [wr.shard_range(S, q, world) for q in range(world)]
    lo, hi = blk[rank]
    # the rank's Bellman-Ford block (oracle rows)
    rows = oracle.bf_many(g, sources[lo:hi], nthreads=2)

    def owned(st, q):
        a, b = blk[q]
        idx = [i for i, v in enumerate(st) if a <= row[int(v)] < b]
        return (idx[0], idx[-1] + 1) if idx else (0, 0)

    counts = np.array([[(owned(st, q)[1] - owned(st, q)[0]) * st.size for st in stops] for q in range(world)])
    offs = np.zeros((world, B + 1), dtype=np.int64)
    offs[:, 1:] = np.cumsum(counts, axis=1)
    max_send = int(offs[:, -1].max())
    send = np.zeros(max_send, dtype=np.int32)
    for o, st in enumerate(stops):
        i0, i1 = owned(st, rank)
        for i in range(i0, i1):
            r = row[int(st[i])] - lo
            send[offs[rank, o] + (i - i0) * st.size: offs[rank, o] + (i - i0 + 1) * st.size] = rows[r, st]
    gathered = torch.zeros(world * max_send, dtype=torch.int32)
    dist.all_gather_into_tensor(gathered, torch.from_numpy(send))
    gathered = gathered.numpy()
    o_lo, o_hi = wr.shard_range(B, rank, world)
    mine = []
    for o in range(o_lo, o_hi):
        st = stops[o]
        n = st.size
        D = np.zeros((n, n), dtype=np.int32)
        for i in range(n):
            q = next(q for q in range(world) if blk[q][0] <= row[int(st[i])] < blk[q][1])
            i0, _ = owned(st, q)
            base = q * max_send + offs[q, o] + (i - i0) * n
            D[i] = gathered[base: base + n]
        c, r, s = oracle.exact_route(D)
        mine.append((o, int(c), int(r), st[s].tolist()))
    objs = [None] * world
    dist.all_gather_object(objs, mine)
    if rank == 0:
        flat = sorted(x for part in objs for x in part)
        ref = oracle.route_orders(g, orders, m=1, nthreads=2)
        ok = all(ref["cost"][o] == c and ref["rank"][o] == r and ref["seq"][o][:len(s)].tolist() == s
                 for o, c, r, s in flat) and len(flat) == B
        with open(out_path, "w") as f:
            f.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_exchange_matches_single(tmp_path, world):
    out = tmp_path / "result.txt"
    mp.spawn(rank_main, args=(world, free_port(), str(out)), nprocs=world, join=True)
    assert out.read_text() == "ok"
