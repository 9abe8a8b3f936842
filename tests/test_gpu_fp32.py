"""GPU: the FP32 variant of the hot path (Tables 9-10).

The FP32 build is the same kernels compiled with Real = float (csrc/hot.cuh); the
oracle stays fp64, so parity here is a rounding bound, not 1e-10.  Derivation of
the bar (reading R27): fp32 unit roundoff u = 6.0e-8; one step
stores Q once per S2O4 stage (2 roundings of ~|Q|) and adds dt*L, whose own
relative error is a few hundred u (LSQ sums over <= 40 members, 50-value records,
~4e3 flops per flux point) but is scaled by dt/h * |F| ~ CFL 0.3; ten steps
accumulate at most ~10 * (2 + 0.3 * 300) u ~ 6e-5 worst case, ~1e-6 typical
(random-walk).  The bar is 3e-5 per conserved variable, relative to max |Q_v|.
The accuracy pin (T7) compares the fp32 and fp64 errors against the exact
solution the way Table 10 does against Table 3.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import hgks, workloads as W

pytestmark = pytest.mark.gpu

TOL32 = 3e-5


def rel_err(a, b):
    """Per-variable max error over the variable's scale.  Momentum components share
    one scale, max_i |rho U_i| (the flux works in rotated face frames, so fp32
    rounding of one component is relative to the whole momentum vector; a component
    that is ~0 everywhere would otherwise divide by ~0).  Reading R27."""
    scale = np.abs(b).max(axis=0)
    scale[1:4] = np.linalg.norm(b[:, 1:4], axis=1).max()
    return np.abs(a - b).max(axis=0) / np.maximum(scale, 1e-300)


EPS32 = 1e-6  # reading R27: the FP32 variant's WENO epsilon; the oracle runs with the same value


def run_pair32(mi, Q0, steps, ocfg=None, gcfg=None):
    ocfg = ocfg or O.OracleConfig(eps=EPS32)
    gcfg = gcfg or hgks.SolverConfig(precision=32)
    assert gcfg.precision == 32 and gcfg.eps_value() == ocfg.eps
    g = hgks.Solver(hgks.Mesh(mi), Q0, gcfg)
    o = O.OracleSolver(O.OracleMesh(mi), Q0, ocfg)
    errs = []
    for _ in range(steps):
        g.step(1)
        o.step(1)
        Qg, gid, tg = g.get_state()
        Qo, to, _, _ = o.state()
        assert np.array_equal(gid, np.arange(mi.n_cells))
        # time bookkeeping is fp64 in both precisions; dt comes from an fp32 state
        assert abs(tg - to) <= 1e-5 * max(1.0, to), (tg, to)
        errs.append(rel_err(Qg, Qo))
    return np.array(errs)


def test_fp32_residual_close_to_oracle(cuda_ok):
    mi = W.kuhn_box(6)
    Q0 = W.advection_ic(mi)
    g = hgks.Solver(hgks.Mesh(mi), Q0, hgks.SolverConfig(precision=32))
    o = O.OracleSolver(O.OracleMesh(mi), Q0, O.OracleConfig(eps=EPS32))
    dt = o.dt()
    Lg, dLg = g.residual(Q0, dt)
    Lo, dLo, _ = o.residual(Q0, dt)
    # L is a difference of O(1) face fluxes divided by V/area ~ 1/h: cancellation
    # costs ~ 1/h * u relative to max|L|
    assert rel_err(Lg, Lo).max() < 1e-4, rel_err(Lg, Lo)
    assert rel_err(dLg, dLo).max() < 1e-4, rel_err(dLg, dLo)


def test_fp32_c1_ten_steps(cuda_ok):
    mi = W.kuhn_box(6)
    errs = run_pair32(mi, W.advection_ic(mi), 10)
    assert errs.max() <= TOL32, errs.max(axis=0)
    assert errs.max() > 0  # really fp32 (fp64 would be ~1e-15)


def test_fp32_jittered_ragged_ten_steps(cuda_ok):
    mi = W.kuhn_box(7, jitter=0.1)
    errs = run_pair32(mi, W.advection_ic(mi), 10)
    assert errs.max() <= TOL32, errs.max(axis=0)


def test_fp32_hex_ns_tau(cuda_ok):
    mi = W.cartesian_hex_box(6, jitter=0.05)
    Q0 = W.random_smooth_ic(mi, seed=118, base=(1.0, 0.3, 0.1, 0.0, 1.0 / 1.4), amp=0.05)
    kw = dict(tau_mode=1, c1=1.0, mu_inf=1e-2, t_inf=1.0 / 1.4, mu_exp=0.7, cfl=0.5)
    errs = run_pair32(mi, Q0, 10, ocfg=O.OracleConfig(eps=EPS32, **kw), gcfg=hgks.SolverConfig(precision=32, **kw))
    assert errs.max() <= TOL32, errs.max(axis=0)


def test_fp32_sphere_wall_farfield(cuda_ok):
    gam, ma, re = 1.4, 0.2535, 118.0
    mi = W.sphere_shell(5)
    fs = (1.0, ma, 0.0, 0.0, 1 / gam)
    Q0 = W.random_smooth_ic(mi, seed=118, base=fs, amp=0.01)
    kw = dict(tau_mode=1, c1=1.0, mu_inf=ma / re, t_inf=1 / gam, mu_exp=0.7, cfl=0.5, freestream=fs)
    errs = run_pair32(mi, Q0, 10, ocfg=O.OracleConfig(eps=EPS32, **kw), gcfg=hgks.SolverConfig(precision=32, **kw))
    assert errs.max() <= TOL32, errs.max(axis=0)


def test_fp32_loopback_ranks_bitwise(cuda_ok):
    """The partitioned fp32 path gives the single-rank fp32 bits (same per-cell arithmetic)."""
    mi = W.kuhn_box(8)
    Q0 = W.advection_ic(mi)
    cfg = hgks.SolverConfig(precision=32)
    ref = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    ref.step(5)
    Qr, _, tr = ref.get_state()
    m2 = hgks.Mesh(mi, n_ranks=3)
    ss = [hgks.Solver(m2, Q0, cfg, rank=r, transport=hgks.TRANSPORT_LOOPBACK) for r in range(3)]
    hgks.group_step(ss, 5)
    Q = np.zeros_like(Qr)
    for s in ss:
        q, gid, t = s.get_state()
        Q[gid] = q
        assert t == tr
    assert np.array_equal(Q, Qr)


def test_fp32_state_memory_halved(cuda_ok):
    mi = W.kuhn_box(8)
    m = hgks.Mesh(mi)
    b64 = m.workspace_size(hgks.SolverConfig())
    b32 = m.workspace_size(hgks.SolverConfig(precision=32))
    # Table 9: FP32 memory ~ 1/2 of FP64 (index arrays stay int32)
    assert 0.5 < b32 / b64 < 0.7, (b32, b64)


def test_precision_validated(cuda_ok):
    mi = W.kuhn_box(6)
    with pytest.raises(hgks.HgksError):
        hgks.Solver(hgks.Mesh(mi), W.advection_ic(mi), hgks.SolverConfig(precision=16))


def _l1_at_t2(N, precision):
    mi = W.kuhn_box(N)
    s = hgks.Solver(hgks.Mesh(mi), W.advection_ic(mi), hgks.SolverConfig(precision=precision))
    while s.step(200, t_stop=2.0)["t"] < 2.0:
        pass
    Q, _, t = s.get_state()
    e = Q[:, 0] - W.advection_ic(mi, t=t)[:, 0]
    s.close()
    return float(np.sum(np.abs(e)) / mi.n_cells)  # uniform volumes: sum |e| V / V_D


def test_fp32_accuracy_table10(cuda_ok):
    """T7 pin (Tables 3 vs 10): FP32 errors deviate from FP64 'slightly'.

    The paper's fp32/fp64 L1 ratios are 1.00006, 1.0004, 1.0023 at N = 10, 20, 40;
    we require |ratio - 1| <= 1e-3, 3e-3, 1e-2 and third order between 20 and 40.
    """
    bars = {10: 1e-3, 20: 3e-3, 40: 1e-2}
    l1 = {}
    for N, bar in bars.items():
        e64, e32 = _l1_at_t2(N, 64), _l1_at_t2(N, 32)
        l1[N] = e32
        assert abs(e32 / e64 - 1) <= bar, (N, e32, e64)
    assert 2.6 <= np.log2(l1[20] / l1[40]) <= 3.3, l1
