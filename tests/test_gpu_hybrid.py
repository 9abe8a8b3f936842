"""GPU parity on hybrid tet/prism meshes (reading R30): the CUDA path
(one mixed-kind layout: 5 faces per cell, triangles and quadrilaterals in separate flux
launches, 6 sub-stencils of up to 7 members with a per-cell count) against the oracle,
with the bar of test_gpu_parity (1e-10 relative after 10 fp64 steps, every step)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import hgks, workloads as W

from test_gpu_parity import TOL, ns_cfgs, rel_err, run_pair

pytestmark = pytest.mark.gpu


def test_hybrid_residual_matches_oracle(cuda_ok):
    mi = W.hybrid_box(6, jitter=0.1)
    Q0 = W.random_smooth_ic(mi, seed=5)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    o = O.OracleSolver(O.OracleMesh(mi), Q0)
    dt = o.dt()
    Lg, dLg = g.residual(Q0, dt)
    Lo, dLo, _ = o.residual(Q0, dt)
    assert rel_err(Lg, Lo).max() < 1e-11, rel_err(Lg, Lo)
    assert rel_err(dLg, dLo).max() < 1e-11, rel_err(dLg, dLo)


def test_hybrid_ten_steps(cuda_ok):
    """Jittered hybrid box (non-planar prism sides), advection, tau = 0."""
    mi = W.hybrid_box(6, jitter=0.1)
    errs, _, _ = run_pair(mi, W.advection_ic(mi), 10)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_hybrid_density_step(cuda_ok):
    """Density step: nonlinear weights far from the linear ones on both cell kinds."""
    mi = W.hybrid_box(6)
    errs, _, _ = run_pair(mi, W.density_step_ic(mi), 10)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_hybrid_ragged_fixed_dt(cuda_ok):
    """7^3 cubes, 3 prism layers: 1470 cells, ragged against the 128-cell tile."""
    mi = W.hybrid_box(7, prism_layers=3)
    Q0 = W.random_smooth_ic(mi, seed=11)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=O.OracleConfig(fixed_dt=2e-3), gcfg=hgks.SolverConfig(fixed_dt=2e-3))
    assert errs.max() <= TOL, errs.max(axis=0)


def test_prisms_only(cuda_ok):
    mi = W.hybrid_box(5, prism_layers=5, jitter=0.05)
    errs, _, _ = run_pair(mi, W.advection_ic(mi), 10)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_hybrid_ns_tau(cuda_ok):
    mi = W.hybrid_box(6, jitter=0.1)
    oc, gc = ns_cfgs(mu=5e-3)
    errs, _, _ = run_pair(mi, W.random_smooth_ic(mi, seed=9), 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


@pytest.mark.parametrize("tau", ["zero", "ns"])
def test_walled_hybrid_box(cuda_ok, tau):
    """Wall faces of both kinds (prism sides and tet faces on the x / y walls)."""
    mi = W.walled_hybrid_box(6, jitter=0.1)
    Q0 = W.random_smooth_ic(mi, seed=7, base=(1.0, 0.3, 0.2, -0.25, 1 / 1.4), amp=0.05)
    if tau == "ns":
        oc, gc = ns_cfgs(mu=1e-2, cfl=0.3)
    else:
        oc, gc = O.OracleConfig(cfl=0.3), hgks.SolverConfig(cfl=0.3)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_hybrid_conservation_free_stream(cuda_ok):
    mi = W.hybrid_box(6, jitter=0.1)
    V = O.OracleMesh(mi).geometry()[0][: mi.n_cells]
    Q0 = W.uniform_state(mi.n_cells, 1.2, (0.4, -0.3, 0.2), 0.9)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    g.step(20)
    Q, _, _ = g.get_state()
    assert np.abs(Q - Q0).max() <= 1e-12 * np.abs(Q0).max()
    Q0 = W.density_step_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    g.step(20)
    Q, _, _ = g.get_state()
    tot0, tot = (Q0 * V[:, None]).sum(0), (Q * V[:, None]).sum(0)
    assert np.abs(tot - tot0).max() <= 1e-13 * np.abs(tot0).max()


@pytest.mark.parametrize("world", [2, 3])
def test_hybrid_multirank_bitwise(cuda_ok, world):
    """Loopback ranks on a hybrid mesh: bitwise equal to the single-rank run."""
    mi = W.hybrid_box(8, jitter=0.1)
    Q0 = W.advection_ic(mi)
    cfg = hgks.SolverConfig(cfl=0.3)
    s1 = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    s1.step(10)
    Q1, _, t1 = s1.get_state()
    mesh = hgks.Mesh(mi, n_ranks=world)
    solvers = [hgks.Solver(mesh, Q0, cfg, rank=r, transport=hgks.TRANSPORT_LOOPBACK) for r in range(world)]
    hgks.group_step(solvers, 10)
    Q = np.empty_like(Q0)
    for s in solvers:
        s.step(0)
        Qr, gid, tr = s.get_state()
        Q[gid] = Qr
        assert tr == t1
    assert np.array_equal(Q, Q1), np.abs(Q - Q1).max()


def test_hybrid_fp32(cuda_ok):
    from test_gpu_fp32 import TOL32, run_pair32
    mi = W.hybrid_box(6, jitter=0.1)
    errs = run_pair32(mi, W.advection_ic(mi), 10)
    assert 0 < errs.max() <= TOL32, errs.max(axis=0)


def hybrid_sphere_case(n, ma, re, prism_layers=None):
    mi = W.sphere_hybrid(n, prism_layers=n // 2 if prism_layers is None else prism_layers)
    gam = 1.4
    fs = (1.0, ma, 0.0, 0.0, 1 / gam)
    Q0 = W.random_smooth_ic(mi, seed=118, base=fs, amp=0.01)
    oc, gc = ns_cfgs(mu=ma / re, c1=1.0, cfl=0.3, fs=fs, t_inf=1 / gam)
    return mi, Q0, oc, gc


@pytest.mark.parametrize("ma,re", [(0.2535, 118.0), (1.5, 300.0)])
def test_hybrid_sphere_wall_farfield(cuda_ok, ma, re):
    """Hybrid tet/prism sphere (prism boundary layer, tets outside; triangle wall and
    farfield faces), NS tau, subsonic and supersonic, 10 steps."""
    mi, Q0, oc, gc = hybrid_sphere_case(4, ma, re)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_c3h_size_steps(cuda_ok):
    """configs[2] as BASELINE.json words it ("~0.5M mixed tet/prism cells"): the hybrid sphere
    at the bench size (N = 20, 10 prism + 30 tet layers, 480,000 cells), parity IC, 10 steps
    (eager step + graph replays), every cell vs the oracle after the first and tenth step."""
    mi, Q0, oc, gc = hybrid_sphere_case(20, 0.2535, 118.0)
    assert mi.n_cells == 480000
    errs, _, _ = run_pair(mi, Q0, 2, ocfg=oc, gcfg=gc, chunks=(1, 9))
    assert errs.max() <= TOL, errs.max(axis=0)
