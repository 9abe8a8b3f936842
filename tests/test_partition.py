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
    if kind == "hybrid":
        return W.hybrid_box(8, jitter=0.1)
    return W.sphere_shell(4)


def put_map_from_tables(plan, rank, tables):
    """The fused-put destinations of rank's send rows from the receivers' (peers, recv_off,
    recv_cnt) tables -- what hgks_p2p_connect does with the tables in the P2P blobs."""
    rr = np.full(plan["send_list"].size, -1, np.int32)
    row = np.full(plan["send_list"].size, -1, np.int32)
    for p, peer in enumerate(plan["peers"]):
        so, sc = int(plan["send_off"][p]), int(plan["send_cnt"][p])
        if not sc:
            continue
        peers_p, off_p, cnt_p = tables[int(peer)]
        k = list(peers_p).index(rank)
        assert cnt_p[k] == sc
        rr[so:so + sc] = peer
        row[so:so + sc] = off_p[k] + np.arange(sc)
    return rr, row


def _worker(rank, world, port, kind, out_q, region=False):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        mi = make_mesh(kind)
        # region=True: this process builds only its own region (hgks_mesh_desc.rank_only)
        mesh = hgks.Mesh(mi, n_ranks=world, rank=rank if region else None)
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
        if region:
            tables = [None] * world
            dist.all_gather_object(tables, (plan["peers"], plan["recv_off"], plan["recv_cnt"]))
            rr, row = put_map_from_tables(plan, rank, tables)
        else:
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


def run_world(world, kind, region=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q, region)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        assert "error" not in v, v.get("error")
    return res


@pytest.mark.parametrize("world,kind", [(2, "kuhn"), (4, "kuhn_jit"), (2, "sphere"), (3, "hybrid")])
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
            for p in range(cf.shape[1]):
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


@pytest.mark.parametrize("world,kind", [(2, "kuhn"), (3, "sphere")])
def test_region_build_exchange_gloo(world, kind):
    """One process per rank, each building only its own region (rank_only, O(owned + ghosts)
    host setup): the plain-RCB partition covers the mesh, every ghost
    arrives bitwise over gloo with the region plans, and the fused-put map built from the
    receivers' exchanged tables (as hgks_p2p_connect builds it) fills every ghost row."""
    res = run_world(world, kind, region=True)
    mi = make_mesh(kind)
    owned = [set(res[r]["owned"]) for r in range(world)]
    assert sum(len(o) for o in owned) == mi.n_cells and len(set().union(*owned)) == mi.n_cells
    for r in range(world):
        assert res[r]["ghosts_ok"], r
        assert res[r]["info"]["edge_cut"] == -1
    # each cut face is counted once on each side
    cut = sum(res[r]["info"]["rank_cut_faces"] for r in range(world))
    assert cut % 2 == 0 and cut > 0


@pytest.mark.parametrize("mk,world", [(lambda: W.kuhn_box(9, jitter=0.1), 3), (lambda: W.sphere_shell(6), 4),
                                      (lambda: W.walled_hex_box(7), 3), (lambda: W.hybrid_box(8, jitter=0.1), 4),
                                      (lambda: W.walled_hybrid_box(7), 3)])
def test_region_plans_equal_whole_mesh_plans(mk, world):
    """A region build gives exactly the plan the whole-mesh build gives for that rank (same
    partition passed in): local ids, peers, send lists, receive ranges and every count."""
    mi = mk()
    whole = hgks.Mesh(mi, n_ranks=world)
    part = np.zeros(mi.n_cells, np.int32)
    for r in range(world):
        p = whole.plan(r)
        part[p["l2g"][:p["n_owned"]]] = r
    whole = hgks.Mesh(mi, n_ranks=world, cell_part=part)
    for r in range(world):
        reg = hgks.Mesh(mi, n_ranks=world, cell_part=part, rank=r)
        a, b = whole.plan(r), reg.plan(r)
        for k in a:
            assert np.array_equal(a[k], b[k]), (r, k)
        ia, ib = whole.info(r), reg.info(r)
        for k in ia:
            if k not in ("edge_cut", "edge_cut_rcb"):
                assert ia[k] == ib[k], (r, k)
        with pytest.raises(hgks.HgksError):
            reg.info((r + 1) % world)


_MEM_SCRIPT = """
import resource, sys
sys.path.insert(0, {root!r})
from paper_2407_00656_b200 import hgks, workloads as W
mi = W.kuhn_box({nx}, {ny}, {nz}, h=2.0 / {nb})
base = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
m = hgks.Mesh(mi, n_ranks={world}, rank={rank})
m.info({r0})
print(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss - base, mi.n_cells)
"""


def test_region_build_host_memory_scales_with_the_rank():
    """Host memory of one rank's setup for the C5 weak-scaling layout (one block per rank,
    here 8 ranks of 24 x 24 x 12 cubes, 41,472 tets each): the region build of rank 0 needs a fraction
    of the whole-mesh build (which holds connectivity for all 8 blocks); peak RSS measured in
    a fresh process per build.  scripts/setup_memory.py reports the full-size C5@8 figures."""
    import subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def peak(rank):
        code = _MEM_SCRIPT.format(root=root, nx=48, ny=48, nz=24, nb=24, world=8, rank=rank,
                                  r0=0)
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr
        kb, n = map(int, out.stdout.split())
        return kb
    whole, region = peak(None), peak(0)
    assert region < 0.35 * whole, (region, whole)
