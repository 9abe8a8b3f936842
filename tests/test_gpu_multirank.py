"""Partitioned GPU path on one B200 via the loopback transport (all ranks in one
process, ghosts exchanged by device copies, min(dt) exact): results must be
BITWISE equal to the single-rank run, and so within the oracle
bar.  The NCCL transport moves the same bytes with the same plans."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import hgks, workloads as W

pytestmark = pytest.mark.gpu


def run_ranks(mi, Q0, cfg, world, steps, t_stop=0.0):
    mesh = hgks.Mesh(mi, n_ranks=world)
    solvers = [hgks.Solver(mesh, Q0, cfg, rank=r, transport=hgks.TRANSPORT_LOOPBACK) for r in range(world)]
    hgks.group_step(solvers, steps, t_stop)
    Q = np.empty_like(Q0)
    t = None
    for s in solvers:
        info = s.step(0)  # sync + positivity check
        Qr, gid, tr = s.get_state()
        Q[gid] = Qr
        t = tr if t is None else t
        assert tr == t
    return Q, t, mesh


@pytest.mark.parametrize("world", [2, 3, 4])
def test_kuhn_multirank_bitwise(cuda_ok, world):
    mi = W.kuhn_box(10, 8, 8, h=0.2)
    Q0 = W.advection_ic(mi)
    cfg = hgks.SolverConfig(cfl=0.3)
    s1 = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    s1.step(10)
    Q1, _, t1 = s1.get_state()
    Qn, tn, mesh = run_ranks(mi, Q0, cfg, world, 10)
    assert tn == t1
    assert np.array_equal(Qn, Q1), np.abs(Qn - Q1).max()
    assert mesh.info(0)["n_peers"] >= 1


@pytest.mark.parametrize("world", [2, 4])
def test_region_meshes_multirank_bitwise(cuda_ok, world):
    """Per-rank region builds (hgks_mesh_desc.rank_only, what each process of a multi-GPU run
    builds): one mesh object per rank, the loopback group's put map assembled from the ranks'
    own plans; 10 steps bitwise equal to one rank (the partition is plain RCB here)."""
    mi = W.kuhn_box(10, 8, 8, h=0.2)
    Q0 = W.advection_ic(mi)
    cfg = hgks.SolverConfig(cfl=0.3)
    s1 = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    s1.step(10)
    Q1, _, t1 = s1.get_state()
    meshes = [hgks.Mesh(mi, n_ranks=world, rank=r) for r in range(world)]
    solvers = [hgks.Solver(meshes[r], Q0, cfg, rank=r, transport=hgks.TRANSPORT_LOOPBACK) for r in range(world)]
    hgks.group_step(solvers, 10)
    Q = np.empty_like(Q0)
    for s in solvers:
        s.step(0)
        Qr, gid, tr = s.get_state()
        Q[gid] = Qr
        assert tr == t1
    assert np.array_equal(Q, Q1), np.abs(Q - Q1).max()


def test_loopback_solver_rejects_plain_step(cuda_ok):
    """A loopback solver of a multi-rank group has no exchange of its own: hgks_step with
    n_steps > 0 fails with HGKS_E_STATE (n_steps = 0, the sync/report call, is allowed)."""
    mi = W.kuhn_box(8)
    mesh = hgks.Mesh(mi, n_ranks=2)
    s = hgks.Solver(mesh, W.advection_ic(mi), hgks.SolverConfig(cfl=0.3), rank=0, transport=hgks.TRANSPORT_LOOPBACK)
    s.step(0)
    with pytest.raises(hgks.HgksError) as e:
        s.step(1)
    assert e.value.code == 7


def test_loopback_fused_put(cuda_ok):
    """f3: the loopback group moves its ghost rows with one k_put per sending rank
    (send rows written straight into the receivers' ghost rows), 2 per step, no
    k_pack; the result stays bitwise equal to one rank (test above)."""
    mi = W.kuhn_box(8)
    Q0 = W.advection_ic(mi)
    mesh = hgks.Mesh(mi, n_ranks=2)
    cfg = hgks.SolverConfig(cfl=0.3)
    solvers = [hgks.Solver(mesh, Q0, cfg, rank=r, transport=hgks.TRANSPORT_LOOPBACK) for r in range(2)]
    for s in solvers:
        s.set_profiling(True)
    hgks.group_step(solvers, 3)
    for r, s in enumerate(solvers):
        s.step(0)
        kt = s.kernel_times()
        assert mesh.info(r)["send_cells"] > 0
        assert kt["k_put"]["launches"] == 6 and "k_pack" not in kt, kt


def test_sphere_multirank_bitwise_and_oracle(cuda_ok):
    mi = W.sphere_shell(5)
    fs = (1.0, 1.5, 0.0, 0.0, 1 / 1.4)
    Q0 = W.random_smooth_ic(mi, seed=118, base=fs, amp=0.01)
    cfg = hgks.SolverConfig(cfl=0.5, tau_mode=1, mu_inf=1.5 / 300, c1=1.0, t_inf=1 / 1.4, freestream=fs)
    s1 = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    s1.step(10)
    Q1, _, t1 = s1.get_state()
    Q4, t4, _ = run_ranks(mi, Q0, cfg, 4, 10)
    assert t4 == t1 and np.array_equal(Q4, Q1)
    oc = O.OracleConfig(cfl=0.5, tau_mode=1, mu_inf=1.5 / 300, c1=1.0, t_inf=1 / 1.4, freestream=fs)
    o = O.OracleSolver(O.OracleMesh(mi), Q0, oc)
    o.step(10)
    Qo, *_ = o.state()
    err = np.abs(Q4 - Qo).max(0) / np.abs(Qo).max(0)
    assert err.max() <= 1e-10, err


def test_multirank_t_stop(cuda_ok):
    mi = W.kuhn_box(8)
    Q0 = W.advection_ic(mi)
    cfg = hgks.SolverConfig(cfl=0.3)
    Q2, t2, _ = run_ranks(mi, Q0, cfg, 2, 50, t_stop=0.04)
    s1 = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    s1.step(50, t_stop=0.04)
    Q1, _, t1 = s1.get_state()
    assert t1 == t2 == 0.04 and np.array_equal(Q1, Q2)


def test_nccl_transport_selftest(cuda_ok):
    """The NCCL calls of a multi-rank step (grouped fp64/fp32 send/recv on a comm
    stream, uint64 allreduce-min on the compute stream) through libhgks's runtime
    NCCL binding, on a one-rank communicator (one GPU here)."""
    hgks.nccl_selftest()


def test_p2p_kernels_selftest(cuda_ok):
    """HGKS_TRANSPORT_P2P's kernels on one device with no cross-rank waiting: k_put via a
    pointer table (bitwise rows, nothing outside them), flag release, acquire-wait on
    flags already set."""
    hgks.p2p_selftest()
