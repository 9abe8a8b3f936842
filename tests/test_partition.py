"""Multi-rank host logic (8(e)) on CPU with world-size 2/4 gloo.

Each rank builds its partition plan through the C-ABI (hgks_mesh_plan) and the
test runs the halo exchange the NCCL path performs -- pack of send_list in plan
order, one message per peer, receive straight into the contiguous ghost range --
over gloo, then checks every ghost against the global field, and checks the
3-layer closure against the oracle's independently built stencils.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2407_00656_b200 import hgks, workloads as W


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_mesh(kind):
    if kind == "kuhn":
        return W.kuhn_box(8, 8, 6, h=0.25)
    if kind == "kuhn_jit":
        return W.kuhn_box(7, jitter=0.1)
    return W.sphere_shell(4)


def _worker(rank, world, port, kind, out_q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        mi = make_mesh(kind)
        mesh = hgks.Mesh(mi, n_ranks=world)
        plan = mesh.plan(rank)
        n_owned = plan["n_owned"]
        l2g = plan["l2g"]
        rng = np.random.default_rng(42)
        Qg = rng.standard_normal((mi.n_cells, 5))        # the global field every rank agrees on
        nl = l2g.size
        Q = np.full((5, nl), np.nan)
        Q[:, :n_owned] = Qg[l2g[:n_owned]].T
        # pack in send_list order (k_pack packs the same rows, 48-byte AoS)
        sl = plan["send_list"]
        ns = sl.size
        buf = Q[:, sl].copy()                              # [5][ns]
        reqs, recv = [], []
        for p, peer in enumerate(plan["peers"]):
            so, sc = plan["send_off"][p], plan["send_cnt"][p]
            if sc:
                msg = torch.from_numpy(np.ascontiguousarray(buf[:, so:so + sc]).ravel())
                reqs.append(dist.isend(msg, int(peer)))
            rc = plan["recv_cnt"][p]
            if rc:
                t = torch.empty(5 * int(rc), dtype=torch.float64)
                reqs.append(dist.irecv(t, int(peer)))
                recv.append((p, t))
        for r in reqs:
            r.wait()
        for p, t in recv:
            ro, rc = plan["recv_off"][p], plan["recv_cnt"][p]
            Q[:, ro:ro + rc] = t.numpy().reshape(5, rc)
        ghosts_ok = bool(np.array_equal(Q.T, Qg[l2g]))
        # fused put (f3): each send row goes to (receiver, ghost row) from hgks_mesh_put_map;
        # emulated as one (rows, values) message per receiver, scattered by the receiver
        rr, row = mesh.put_map(rank)
        Qp = np.full((5, nl), np.nan)
        Qp[:, :n_owned] = Q[:, :n_owned]
        reqs, recv = [], []
        for p, peer in enumerate(plan["peers"]):
            sel = np.nonzero(rr == peer)[0]
            if sel.size:
                reqs.append(dist.isend(torch.from_numpy(row[sel].astype(np.float64)), int(peer)))
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Q[:, sl[sel]]).ravel()), int(peer)))
            rc = int(plan["recv_cnt"][p])
            if rc:
                tr, tv = torch.empty(rc, dtype=torch.float64), torch.empty(5 * rc, dtype=torch.float64)
                reqs.append(dist.irecv(tr, int(peer)))
                reqs.append(dist.irecv(tv, int(peer)))
                recv.append((tr, tv, rc))
        for r in reqs:
            r.wait()
        for tr, tv, rc in recv:
            Qp[:, tr.numpy().astype(np.int64)] = tv.numpy().reshape(5, rc)
        ghosts_ok = ghosts_ok and bool(np.array_equal(Qp.T, Qg[l2g]))
        info = mesh.info(rank)
        out_q.put((rank, dict(owned=l2g[:n_owned].tolist(), ghosts=l2g[n_owned:].tolist(), ghosts_ok=ghosts_ok,
                              info=info, send_total=int(ns))))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        out_q.put((rank, dict(error=traceback.format_exc())))


def run_world(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        assert "error" not in v, v.get("error")
    return res


@pytest.mark.parametrize("world,kind", [(2, "kuhn"), (4, "kuhn_jit"), (2, "sphere")])
def test_partition_exchange_gloo(world, kind):
    res = run_world(world, kind)
    mi = make_mesh(kind)
    owned = [set(res[r]["owned"]) for r in range(world)]
    # owned sets partition the mesh, balanced (RCB: sizes differ by < 1%)
    assert sum(len(o) for o in owned) == mi.n_cells
    assert len(set().union(*owned)) == mi.n_cells
    sizes = np.array([len(o) for o in owned])
    assert sizes.max() - sizes.min() <= max(1, 0.01 * sizes.mean())
    # every ghost value arrived bitwise from its owner
    for r in range(world):
        assert res[r]["ghosts_ok"], r
        info = res[r]["info"]
        assert info["n_ghost"] == len(res[r]["ghosts"])
        # overlap split: some but not all cells/faces need no ghosts
        assert 0 < info["n_early_cells"] < info["n_owned"]
        assert 0 < info["n_early_faces"] < info["n_faces"]
    # send volume of all ranks == receive volume of all ranks
    assert sum(res[r]["send_total"] for r in range(world)) == sum(len(res[r]["ghosts"]) for r in range(world))
    # 3-layer closure against the oracle's independent stencils: every cell the
    # fluxes of an owned cell's faces touch (both sides' big stencils) is local
    om = O.OracleMesh(mi)
    f = om.faces()
    cf = om.cell_faces()
    big = {}

    def stencil(c):
        if c not in big:
            big[c] = set(int(x) for x in om.big_stencil(c)[0] if x < om.n_cells) | {c}
        return big[c]

    for r in range(world):
        local = owned[r] | set(res[r]["ghosts"])
        for c in list(owned[r])[::3]:
            for p in range(6):
                fi = cf[c, p]
                if fi < 0:
                    continue
                for side in (f["owner"][fi], f["nb"][fi]):
                    if side >= 0:
                        assert stencil(int(side)) <= local, (r, c, side)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_put_map_is_a_bijection_onto_ghost_rows(world):
    """hgks_mesh_put_map (f3): every send row of every rank lands on a ghost row of its
    receiver holding the same global cell, and every ghost row of every rank is written
    exactly once (host plans only; the loopback GPU tests run k_put with these maps)."""
    mi = W.kuhn_box(8, 8, 6, h=0.25)
    mesh = hgks.Mesh(mi, n_ranks=world)
    plans = [mesh.plan(r) for r in range(world)]
    hits = [np.zeros(p["l2g"].size, np.int64) for p in plans]
    for q in range(world):
        rr, row = mesh.put_map(q)
        sl = plans[q]["send_list"]
        assert rr.size == sl.size
        for p in set(rr.tolist()):
            sel = rr == p
            assert p != q and p in plans[q]["peers"]
            assert np.all(row[sel] >= plans[p]["n_owned"])
            assert np.array_equal(plans[p]["l2g"][row[sel]], plans[q]["l2g"][sl[sel]])
            np.add.at(hits[p], row[sel], 1)
    for p in range(world):
        n_owned = plans[p]["n_owned"]
        assert np.all(hits[p][:n_owned] == 0) and np.all(hits[p][n_owned:] == 1), p
