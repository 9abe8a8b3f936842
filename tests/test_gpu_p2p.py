"""HGKS_TRANSPORT_P2P across processes, one GPU per rank: the fused
NVLink put with per-stage epoch flags must give results bitwise equal to one rank and
to the NCCL transport.  Needs >= 2 GPUs on one node; skipped otherwise (every gpurun
box has one GPU, so this runs first on a multi-GPU node)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, transport, out_q):
    try:
        import torch.distributed as dist
        from paper_2407_00656_b200 import hgks, workloads as W
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        mi = W.kuhn_box(10, 8, 8, h=0.2)
        Q0 = W.advection_ic(mi)
        mesh = hgks.Mesh(mi, n_ranks=world)
        obj = [hgks.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        tr = hgks.TRANSPORT_P2P if transport == "p2p" else hgks.TRANSPORT_NCCL
        s = hgks.Solver(mesh, Q0, hgks.SolverConfig(cfl=0.3), device=rank, rank=rank, nccl_id=obj[0], transport=tr)
        if tr == hgks.TRANSPORT_P2P:
            s.p2p_connect_dist()
        s.step(10)
        Q, gid, t = s.get_state()
        out_q.put((rank, dict(Q=Q, gid=gid, t=t)))
        dist.barrier()
        s.close()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        out_q.put((rank, dict(error=traceback.format_exc())))


def _run(transport):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, transport, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    for v in res.values():
        assert "error" not in v, v["error"]
    return res


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < WORLD,
                    reason="needs >= 2 GPUs on one node")
def test_p2p_transport_bitwise_equals_one_rank_and_nccl():
    from paper_2407_00656_b200 import hgks, workloads as W
    mi = W.kuhn_box(10, 8, 8, h=0.2)
    Q0 = W.advection_ic(mi)
    s1 = hgks.Solver(hgks.Mesh(mi), Q0, hgks.SolverConfig(cfl=0.3))
    s1.step(10)
    Q1, _, t1 = s1.get_state()
    for transport in ("p2p", "nccl"):
        res = _run(transport)
        Q = np.empty_like(Q1)
        for v in res.values():
            Q[v["gid"]] = v["Q"]
            assert v["t"] == t1
        assert np.array_equal(Q, Q1), (transport, np.abs(Q - Q1).max())
