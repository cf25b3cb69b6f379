"""a9 in separate processes: libwr's sharded phases (wr_orders_plan /
wr_orders_local / wr_orders_finish) run in two processes on one GPU, the
send buffers exchanged by a gloo all-gather of host-staged copies (the
layout torch.distributed.all_gather_into_tensor produces over NCCL), and
the concatenated results compared with the CPU oracle. No kernel waits on
another process: each rank's kernels finish before its host copy, so two
processes sharing one GPU is safe (B200_PROFILING.md). The N>1 bench runs
the same phases with NCCL on separate GPUs."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, cfg, B, wtype, m, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import gen
    import paper_2504_20655_b200 as wr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g, orders, _ = gen.config(cfg, wtype=wtype, B=B)
    G = wr.Graph.from_gen(g, device=0)
    p = wr.OrdersPlan(G, orders.order_ptr, orders.order_nodes, rank, world, m=m)
    info = p.info
    send = torch.zeros(info.max_send, dtype=torch.int32, device="cuda")
    p.local(send)
    torch.cuda.synchronize()
    parts = [torch.empty(info.max_send, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(parts, send.cpu())
    gathered = torch.cat(parts).cuda()
    res, _ = p.finish(gathered)
    np.save(os.path.join(out, f"r{rank}.npy"), res)
    p.close()
    G.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,B,wtype,m", [(3, 1200, "i32", 1), (3, 600, "f32", 1), (4, 96, "i32", 3)])
def test_sharded_phases_two_processes_vs_oracle(tmp_path, cfg, B, wtype, m):
    import torch.multiprocessing as mp

    import gen
    import oracle
    import paper_2504_20655_b200 as wr

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    world = 2
    mp.start_processes(_rank, args=(world, _port(), cfg, B, wtype, m, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)])
    g, orders, _ = gen.config(cfg, wtype=wtype, B=B)
    exp = oracle.route_orders(g, orders, m=m)
    assert got.shape[0] == orders.B
    ok = exp["order_rc"] == 0
    assert ok.all()
    assert (got["status"] == 0).all()
    cost = wr.decode_cost(got, wr.WR_F32 if wtype == "f32" else wr.WR_I32)
    assert cost.tobytes() == exp["cost"].tobytes()
    assert np.array_equal(got["seq"], exp["seq"]) and np.array_equal(got["rank"], exp["rank"])
