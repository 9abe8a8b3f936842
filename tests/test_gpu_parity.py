"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star; reading R26): after 10 fp64 steps, per conserved
variable v, max_i |Q_gpu - Q_oracle| / max_i |Q_oracle| <= 1e-10.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import hgks, workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel_err(a, b):
    return (np.abs(a - b).max(axis=0) / np.maximum(np.abs(b).max(axis=0), 1e-300))


def run_pair(mi, Q0, steps, cfl=0.3, per_step=True, ocfg=None, gcfg=None, chunks=None):
    """Advance the CUDA path and the oracle side by side and compare after every chunk of
    steps (default: every step)."""
    ocfg = ocfg or O.OracleConfig(cfl=cfl)
    gcfg = gcfg or hgks.SolverConfig(cfl=cfl)
    g = hgks.Solver(hgks.Mesh(mi), Q0, gcfg)
    o = O.OracleSolver(O.OracleMesh(mi), Q0, ocfg)
    errs = []
    if chunks is None:
        chunks = [1] * steps if per_step else [steps]
    for n in chunks:
        gi = g.step(n)
        o.step(n)
        Qg, gid, tg = g.get_state()
        Qo, to, dto, fbo = o.state()
        assert np.array_equal(gid, np.arange(mi.n_cells))
        assert abs(tg - to) <= 1e-13 * max(1.0, to), (tg, to)
        assert gi["fallbacks"] == fbo
        errs.append(rel_err(Qg, Qo))
    return np.array(errs), g, o


def gpu_and_oracle(mi, Q0, gcfg, ocfg, steps):
    """Full-size runs: the oracle (mesh build + steps on all host cores) in a worker thread
    while the CUDA path builds its mesh and steps (ctypes releases the GIL), so the test
    takes about the oracle's time alone.  Returns (Q_gpu, t_gpu, oracle state)."""
    from concurrent.futures import ThreadPoolExecutor

    def oracle_run():
        o = O.OracleSolver(O.OracleMesh(mi), Q0, ocfg)
        o.step(steps)
        return o.state()

    with ThreadPoolExecutor(1) as ex:
        fut = ex.submit(oracle_run)
        g = hgks.Solver(hgks.Mesh(mi), Q0, gcfg)
        g.step(steps)
        Qg, _, tg = g.get_state()
        del g
        return Qg, tg, fut.result()


def test_c1_residual_matches_oracle(cuda_ok):
    mi = W.kuhn_box(6)
    Q0 = W.advection_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    o = O.OracleSolver(O.OracleMesh(mi), Q0)
    dt = o.dt()
    Lg, dLg = g.residual(Q0, dt)
    Lo, dLo, _ = o.residual(Q0, dt)
    assert rel_err(Lg, Lo).max() < 1e-11, rel_err(Lg, Lo)
    assert rel_err(dLg, dLo).max() < 1e-11, rel_err(dLg, dLo)


def test_c1_ten_steps(cuda_ok):
    """C1: 1296 Kuhn tets, periodic [0,2]^3, tau = 0, CFL 0.3, 10 steps, every step."""
    mi = W.kuhn_box(6)
    errs, _, _ = run_pair(mi, W.advection_ic(mi), 10)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_jittered_tets_ten_steps(cuda_ok):
    mi = W.kuhn_box(6, jitter=0.1)
    Q0 = W.advection_ic(mi)
    errs, _, _ = run_pair(mi, Q0, 10)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_ragged_box_fixed_dt(cuda_ok):
    """Non-cubic box (7x5x6 cubes, ragged against every tile size), fixed dt."""
    mi = W.kuhn_box(7, 5, 6, h=2.0 / 6)
    Q0 = W.random_smooth_ic(mi, seed=7)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=O.OracleConfig(fixed_dt=2e-3), gcfg=hgks.SolverConfig(fixed_dt=2e-3))
    assert errs.max() <= TOL, errs.max(axis=0)


def test_hex_box_ten_steps(cuda_ok):
    mi = W.cartesian_hex_box(6, jitter=0.1)
    Q0 = W.random_smooth_ic(mi, seed=3)
    errs, _, _ = run_pair(mi, Q0, 10, cfl=0.5)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_stress_step_density(cuda_ok):
    """C1s-like (tau = 0 variant): density step, nonlinear weights far from gamma."""
    mi = W.kuhn_box(6)
    Q0 = W.density_step_ic(mi)
    errs, _, _ = run_pair(mi, Q0, 10)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_t_stop_clipping(cuda_ok):
    mi = W.kuhn_box(6)
    Q0 = W.advection_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    o = O.OracleSolver(O.OracleMesh(mi), Q0)
    info = g.step(100, t_stop=0.05)
    o.step(100, 0.05)
    Qo, to, _, _ = o.state()
    Qg, _, tg = g.get_state()
    assert tg == 0.05 and to == 0.05
    assert rel_err(Qg, Qo).max() <= TOL
    assert g.step(5, t_stop=0.05)["steps_done"] == 0


def test_positivity_fallbacks_fire_and_match(cuda_ok):
    """R21 with fallbacks > 0: one cell of density and pressure x1000 in a uniform flow on the
    C1 mesh (tau = 0 and NS tau); 10 steps, the GPU's cumulative fallback count equals the
    oracle's after every step and the state meets the bar."""
    mi = W.kuhn_box(6)
    for oc, gc in ((O.OracleConfig(cfl=0.3), hgks.SolverConfig(cfl=0.3)), ns_cfgs(mu=1e-3)):
        errs, g, o = run_pair(mi, W.spike_state(mi), 10, ocfg=oc, gcfg=gc)
        assert o.state()[3] > 0
        assert errs.max() <= TOL, errs.max(axis=0)


def test_t_stop_ns_tau_steps_after_stop(cuda_ok):
    """NS tau (moment form, 1/dt in the time fit) with t_stop: the steps requested after
    t reached t_stop have dt = 0 and leave the state unchanged (no 0 * inf)."""
    mi = W.kuhn_box(6)
    oc, gc = ns_cfgs(mu=1e-3)
    Q0 = W.density_step_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0, gc)
    o = O.OracleSolver(O.OracleMesh(mi), Q0, oc)
    info = g.step(50, t_stop=0.02)
    o.step(50, 0.02)
    assert info["t"] == 0.02 and 0 < info["steps_done"] < 50
    Qo, to, _, _ = o.state()
    Qg, _, tg = g.get_state()
    assert tg == to == 0.02
    assert rel_err(Qg, Qo).max() <= TOL
    assert g.step(3, t_stop=0.02)["steps_done"] == 0
    Qg2, _, _ = g.get_state()
    assert np.array_equal(Qg, Qg2)


def test_bench_size_steps(cuda_ok):
    """configs[1] at its top size N=48 (663,552 tets) for 10 steps in bench.py's launch
    configuration (one eager step, then CUDA-graph replays): every cell vs the oracle after
    the first step and after the tenth."""
    mi = W.kuhn_box(48)
    Q0 = W.advection_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0, hgks.SolverConfig(cfl=0.3))
    o = O.OracleSolver(O.OracleMesh(mi), Q0, O.OracleConfig(cfl=0.3))
    for n in (1, 9):
        gi = g.step(n)
        o.step(n)
        Qg, _, tg = g.get_state()
        Qo, to, _, fbo = o.state()
        assert abs(tg - to) <= 1e-13 and gi["fallbacks"] == fbo == 0
        assert rel_err(Qg, Qo).max() <= TOL, rel_err(Qg, Qo)


def test_c5_full_size_two_steps(cuda_ok):
    """configs[4] at full size: the 110^3 Kuhn box (7,986,000 tets, bench.py's default
    workload) for 2 steps in the bench launch configuration (eager step + graph replay),
    every cell vs the oracle (all host cores; SURVEY 8(d) C5 allows >= 2 oracle steps)."""
    mi = W.kuhn_box(110)
    Q0 = W.advection_ic(mi)
    Qg, tg, (Qo, to, _, fbo) = gpu_and_oracle(mi, Q0, hgks.SolverConfig(cfl=0.3), O.OracleConfig(cfl=0.3), 2)
    assert abs(tg - to) <= 1e-13 and fbo == 0
    assert rel_err(Qg, Qo).max() <= TOL, rel_err(Qg, Qo)


def test_conservation_and_free_stream_gpu(cuda_ok):
    mi = W.kuhn_box(8, jitter=0.1)
    V = O.OracleMesh(mi).geometry()[0][: mi.n_cells]
    Q0 = W.uniform_state(mi.n_cells, 1.0, (0.3, -0.2, 0.5), 1.0)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    g.step(20)
    Q, _, _ = g.get_state()
    assert np.abs(Q - Q0).max() <= 1e-12
    Q0 = W.advection_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0)
    g.step(20)
    Q, _, _ = g.get_state()
    tot0 = (Q0 * V[:, None]).sum(0)
    tot = (Q * V[:, None]).sum(0)
    assert np.abs(tot - tot0).max() <= 1e-12 * np.abs(tot0).max()


# --------------------------------------------------------------------------- #
# tau > 0 (Navier-Stokes collision time, moment form) and boundary faces
# --------------------------------------------------------------------------- #
def ns_cfgs(mu=1e-3, c1=1.0, cfl=0.3, fs=(1.0, 0.0, 0.0, 0.0, 1 / 1.4), t_inf=1.0):
    o = O.OracleConfig(cfl=cfl, tau_mode=1, mu_inf=mu, c1=c1, t_inf=t_inf, freestream=fs)
    g = hgks.SolverConfig(cfl=cfl, tau_mode=1, mu_inf=mu, c1=c1, t_inf=t_inf, freestream=fs)
    return o, g


def test_c1s_stress_ns_tau(cuda_ok):
    """C1s: density step, tau = mu/p + C1 |pl-pr|/(pl+pr) dt (R7), 10 steps."""
    mi = W.kuhn_box(6)
    oc, gc = ns_cfgs()
    errs, _, _ = run_pair(mi, W.density_step_ic(mi), 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_hex_box_ns_tau(cuda_ok):
    mi = W.cartesian_hex_box(6, jitter=0.1)
    oc, gc = ns_cfgs(mu=5e-3, cfl=0.5)
    errs, _, _ = run_pair(mi, W.random_smooth_ic(mi, seed=9), 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


@pytest.mark.parametrize("tau", ["zero", "ns"])
def test_walled_box(cuda_ok, tau):
    """Closed box, six wall sides (R25 mirror ghosts; cells with 1, 2 and 3 wall
    faces), jittered interior nodes: 10 steps, tau = 0 (Euler-chain flux with wall
    faces) and NS tau (moment form)."""
    mi = W.walled_hex_box(6, h=0.4, jitter=0.1)
    Q0 = W.random_smooth_ic(mi, seed=7, base=(1.0, 0.3, 0.2, -0.25, 1 / 1.4), amp=0.05)
    if tau == "ns":
        oc, gc = ns_cfgs(mu=1e-2, cfl=0.5)
    else:
        oc, gc = O.OracleConfig(cfl=0.5), hgks.SolverConfig(cfl=0.5)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


def sphere_case(n, ma, re):
    mi = W.sphere_shell(n)
    gam = 1.4
    fs = (1.0, ma, 0.0, 0.0, 1 / gam)
    # SURVEY 8(d) parity IC: free stream x (1 + 0.01 sum sin) on rho and p
    Q0 = W.random_smooth_ic(mi, seed=118, base=fs, amp=0.01)
    oc, gc = ns_cfgs(mu=ma * 1.0 / re, c1=1.0, cfl=0.5, fs=fs, t_inf=1 / gam)
    return mi, Q0, oc, gc


def test_sphere_subsonic_wall_farfield(cuda_ok):
    """C3 parity at small N: hex sphere shell, Ma 0.2535, Re 118, wall + farfield faces."""
    mi, Q0, oc, gc = sphere_case(5, 0.2535, 118.0)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_sphere_supersonic_wall_farfield(cuda_ok):
    """C4 parity at small N: Ma 1.5, Re 300 (supersonic inflow/outflow farfield faces)."""
    mi, Q0, oc, gc = sphere_case(4, 1.5, 300.0)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


def test_sphere_residual_matches_oracle(cuda_ok):
    mi, Q0, oc, gc = sphere_case(4, 0.2535, 118.0)
    g = hgks.Solver(hgks.Mesh(mi), Q0, gc)
    o = O.OracleSolver(O.OracleMesh(mi), Q0, oc)
    dt = o.dt()
    Lg, dLg = g.residual(Q0, dt)
    Lo, dLo, _ = o.residual(Q0, dt)
    # moment form with tau ~ dt: the time-integral coefficients cancel to O(dt^3/tau)
    # (SURVEY A.3), so intermediates carry ~1e-11; the 10-step state bar stays 1e-10
    assert rel_err(Lg, Lo).max() < 1e-10, rel_err(Lg, Lo)
    assert rel_err(dLg, dLo).max() < 1e-10, rel_err(dLg, dLo)


def test_pipelined_host_io_matches_synchronous(cuda_ok):
    """hgks_set_state / hgks_get_state_async / hgks_sync (copies on the library's own
    streams, double-buffered) give the same bits as the synchronous calls."""
    import torch
    mi = W.kuhn_box(7, jitter=0.1)
    Q0 = W.advection_ic(mi)
    a = hgks.Solver(hgks.Mesh(mi), Q0)
    b = hgks.Solver(hgks.Mesh(mi), Q0)
    outs = [torch.zeros((mi.n_cells, 5), dtype=torch.float64).pin_memory() for _ in range(2)]
    ref = []
    Qin = torch.from_numpy(Q0.copy()).pin_memory()
    for k in range(5):
        a.set_state(Q0, 0.0)
        a.step(k + 1)
        ref.append(a.get_state()[0])
    for k in range(5):
        b.set_state(Qin, 0.0)
        b.step(k + 1, info=False)
        b.get_state_async(outs[k % 2])
        if k % 2 == 1:
            b.sync()
            assert np.array_equal(outs[0].numpy(), ref[k - 1])
            assert np.array_equal(outs[1].numpy(), ref[k])
    b.sync()
    assert np.array_equal(outs[0].numpy(), ref[4])


def test_cuda_graph_steps_match_eager(cuda_ok, monkeypatch):
    """hgks_step replays a captured CUDA graph of one step (single rank): same bits as
    eager launches, including t_stop clipping (the graph is re-captured per t_stop)."""
    mi = W.kuhn_box(7, jitter=0.1)
    Q0 = W.advection_ic(mi)
    out = {}
    for g in ("0", "1"):
        monkeypatch.setenv("HGKS_GRAPHS", g)
        s = hgks.Solver(hgks.Mesh(mi), Q0)
        s.step(1)
        s.step(6)
        s.step(5, t_stop=0.08)
        out[g] = s.get_state()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert out["0"][2] == out["1"][2]


def test_c3_size_steps(cuda_ok):
    """configs[2] at the bench size (sphere shell N = 35, 514,500 hexes; NS tau, wall +
    farfield) with the parity IC for 10 steps (eager step + graph replays), every cell vs
    the oracle after the first and the tenth step."""
    mi, Q0, oc, gc = sphere_case(35, 0.2535, 118.0)
    errs, _, _ = run_pair(mi, Q0, 2, ocfg=oc, gcfg=gc, chunks=(1, 9))
    assert errs.max() <= TOL, errs.max(axis=0)


def test_c4_full_size_two_steps(cuda_ok):
    """configs[3] at full size (sphere shell N = 70, 4,116,000 hexes, Ma 1.5, Re 300: the
    supersonic farfield states) with the parity IC, 2 steps, every cell vs the oracle."""
    mi, Q0, oc, gc = sphere_case(70, 1.5, 300.0)
    Qg, tg, (Qo, to, _, fbo) = gpu_and_oracle(mi, Q0, gc, oc, 2)
    assert abs(tg - to) <= 1e-13 * max(1.0, to)
    assert rel_err(Qg, Qo).max() <= TOL, rel_err(Qg, Qo)


@pytest.mark.parametrize("pair", ["0", "1"])
def test_recon_lane_pair_variant(cuda_ok, monkeypatch, pair):
    """Reconstruction with one or two lanes per cell (the fp32 default is two) meets the bar
    on the jittered tet box and the sphere shell."""
    monkeypatch.setenv("HGKS_RECON_PAIR", pair)
    mi = W.kuhn_box(7, jitter=0.1)
    errs, _, _ = run_pair(mi, W.advection_ic(mi), 5)
    assert errs.max() <= TOL, errs.max(axis=0)
    mi, Q0, oc, gc = sphere_case(4, 0.2535, 118.0)
    errs, _, _ = run_pair(mi, Q0, 5, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)


@pytest.mark.parametrize("mode", [1, 2])
def test_dq0_readings_match_oracle(cuda_ok, mode):
    """SURVEY Q9 readings of dQ0 (R9k kinetic weighting, R9s linear-weight gradients) in both
    flux forms: C1 (tau = 0), the fallback stress state (NS tau, fallbacks > 0) and the sphere
    shell (wall + farfield faces, NS tau); 10 steps each within the bar."""
    mi = W.kuhn_box(6)
    errs, _, _ = run_pair(mi, W.advection_ic(mi), 10, ocfg=O.OracleConfig(dq0_mode=mode),
                          gcfg=hgks.SolverConfig(dq0_mode=mode))
    assert errs.max() <= TOL, errs.max(axis=0)
    oc, gc = ns_cfgs(mu=1e-3)
    oc.dq0_mode = gc.dq0_mode = mode
    errs, _, o = run_pair(mi, W.spike_state(mi), 10, ocfg=oc, gcfg=gc)
    assert o.state()[3] > 0
    assert errs.max() <= TOL, errs.max(axis=0)
    mi, Q0, oc, gc = sphere_case(4, 0.2535, 118.0)
    oc.dq0_mode = gc.dq0_mode = mode
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)
    mi = W.walled_hex_box(6, h=0.4, jitter=0.1)  # tau = 0 with wall faces
    Q0 = W.random_smooth_ic(mi, seed=7, base=(1.0, 0.3, 0.2, -0.25, 1 / 1.4), amp=0.05)
    errs, _, _ = run_pair(mi, Q0, 10, ocfg=O.OracleConfig(cfl=0.5, dq0_mode=mode),
                          gcfg=hgks.SolverConfig(cfl=0.5, dq0_mode=mode))
    assert errs.max() <= TOL, errs.max(axis=0)


def test_prandtl_fix_matches_oracle(cuda_ok):
    """R29 heat-flux correction at Pr = 0.72 (moment form): the C1s stress state with NS tau
    and the sphere shell (wall + farfield, the viscous sphere of P:1203-1210) for 10 steps
    within the bar; tau = 0 is unaffected by construction (checked on the oracle side)."""
    mi = W.kuhn_box(6)
    oc, gc = ns_cfgs(mu=1e-3)
    oc.prandtl = gc.prandtl = 0.72
    errs, _, _ = run_pair(mi, W.density_step_ic(mi), 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)
    mi, Q0, oc, gc = sphere_case(4, 0.2535, 118.0)
    oc.prandtl = gc.prandtl = 0.72
    errs, g, _ = run_pair(mi, Q0, 10, ocfg=oc, gcfg=gc)
    assert errs.max() <= TOL, errs.max(axis=0)
    # the fix changes the solution (it is not a no-op on this viscous case)
    oc1, gc1 = sphere_case(4, 0.2535, 118.0)[2:]
    g1 = hgks.Solver(hgks.Mesh(mi), Q0, gc1)
    g1.step(10)
    assert np.abs(g1.get_state()[0] - g.get_state()[0]).max() > 1e-9
