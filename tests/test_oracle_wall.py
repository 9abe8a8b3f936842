"""Oracle pins for the wall boundary (R25: mirror ghost, all velocity components
reversed, normal derivatives negated; Alg. 1 "Add ghost cell according to boundary
condition"; adiabatic no-slip sphere surface).

A closed box whose six sides are all walls: interior faces cancel exactly in
sum_i V_i L_i, so the totals are the wall-face fluxes alone (L_i = -(1/V_i) sum_f s F S,
P:240-244).  What the mathematics fixes there, independently of the oracle's code:
* tau = 0: the mirror pair's equilibrium state Q0 (compatibility) is at
  rest, so the wall passes no mass and no energy, and neither does d_t F (Euler chain,
  SURVEY A.10): sum V L and sum V d_t L vanish in those components to round-off;
* tau = 0: the wall momentum flux is the stagnation pressure p0 n with
  p0 = (gamma-1) rho [U m1 + m0 (V^2 + W^2) + m0 (K+3)/(2 lam)], m0, m1 the textbook
  half-range Maxwellian moments (erfc / exp closed forms) of the owner's Gauss-point
  state -- the tangential kinetic energy turns into pressure only for a no-slip mirror,
  so a slip mirror fails this;
* any tau: the wall faces inside residual() equal the Gauss-point flux of the mirror
  pair built here from R25's definition.
"""
import numpy as np
import pytest
from scipy.special import erfc

from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W


def _setup(tau_mode):
    mi = W.walled_hex_box(5, h=0.4)
    Q = W.random_smooth_ic(mi, seed=7, base=(1.0, 0.3, 0.2, -0.25, 1 / 1.4), amp=0.05)
    cfg = O.OracleConfig(tau_mode=tau_mode, mu_inf=0.01, c1=1.0, t_inf=1 / 1.4)
    m = O.OracleMesh(mi)
    s = O.OracleSolver(m, Q, cfg)
    dt = s.dt()
    L, dL, fb = s.residual(Q, dt)
    assert fb == 0
    V = m.geometry()[0][:mi.n_cells]
    return mi, Q, cfg, m, dt, (V[:, None] * L).sum(0), (V[:, None] * dL).sum(0), (V[:, None] * np.abs(L)).sum(0)


def _wall_totals(m, Q, cfg, dt, mode):
    """-sum over wall Gauss points of omega S F (global frame) for the expected F."""
    fc = m.faces()
    g, K = cfg.gamma, cfg.K
    sv = np.array([1.0, -1.0, -1.0, -1.0, 1.0])
    tot, totd = np.zeros(5), np.zeros(5)
    for f in np.nonzero(fc["bc"] == W.BC_WALL)[0]:
        ng = fc["ngp"][f]
        val, grad = m.weno_points(Q, fc["owner"][f], fc["gp_x"][f, :ng], cfg)
        for k in range(ng):
            n = fc["gp_n"][f, k]
            t1, t2 = O.local_frame(n)
            R = np.array([n, t1, t2])
            v5 = val[k]
            if mode == "closed":
                rho = v5[0]
                u = R @ v5[1:4] / rho
                p = (g - 1) * (v5[4] - 0.5 * rho * (u @ u))
                lam, U = rho / (2 * p), u[0]
                m0 = 0.5 * erfc(-np.sqrt(lam) * U)
                m1 = U * m0 + np.exp(-lam * U * U) / (2 * np.sqrt(np.pi * lam))
                E0 = rho * (U * m1 + m0 * (u[1] ** 2 + u[2] ** 2) + m0 * (K + 3) / (2 * lam))
                F, dF = np.array([0.0, (g - 1) * E0, 0.0, 0.0, 0.0]), np.zeros(5)
            elif mode == "slip":  # what a slip mirror (tangential velocity kept) would give
                rho = v5[0]
                u = R @ v5[1:4] / rho
                p = (g - 1) * (v5[4] - 0.5 * rho * (u @ u))
                lam, U = rho / (2 * p), u[0]
                m0 = 0.5 * erfc(-np.sqrt(lam) * U)
                m1 = U * m0 + np.exp(-lam * U * U) / (2 * np.sqrt(np.pi * lam))
                F, dF = np.array([0.0, (g - 1) * rho * (U * m1 + m0 * (K + 3) / (2 * lam)), 0.0, 0.0, 0.0]), np.zeros(5)
            else:  # the mirror pair of R25, flux by the Gauss-point routine
                ql = np.r_[v5[0], R @ v5[1:4], v5[4]]
                dql = np.zeros((3, 5))
                for j in range(3):
                    d = grad[k] @ R[j]
                    dql[j] = np.r_[d[0], R @ d[1:4], d[4]]
                dqr = np.array([-sv * dql[0], sv * dql[1], sv * dql[2]])
                o = O.gp_flux(ql, dql, sv * ql, dqr, dt, cfg)
                F, dF = o["F"], o["dF"]
            w = fc["gp_wS"][f, k]
            for a, b in ((F, tot), (dF, totd)):
                b[0] -= w * a[0]
                b[4] -= w * a[4]
                b[1:4] -= w * (R.T @ a[1:4])
    return tot, totd


def test_wall_is_impermeable_and_adiabatic_tau0():
    *_, tot, totd, scale = _setup(0)
    for v in (0, 4):
        assert abs(tot[v]) <= 1e-14 * scale[v], (v, tot, scale)
        assert abs(totd[v]) <= 1e-14 * scale[v], (v, totd, scale)
    assert np.abs(tot[1:4]).max() > 0.1  # the walls do push (momentum is not conserved)


def test_wall_stagnation_pressure_closed_form_tau0():
    mi, Q, cfg, m, dt, tot, totd, scale = _setup(0)
    exp, _ = _wall_totals(m, Q, cfg, dt, "closed")
    assert np.abs(tot - exp).max() <= 1e-13 * scale.max(), (tot, exp)
    slip, _ = _wall_totals(m, Q, cfg, dt, "slip")
    assert np.abs(tot[1:4] - slip[1:4]).max() > 1e-3  # the pin tells no-slip from slip


@pytest.mark.parametrize("tau_mode", [0, 1])
def test_wall_faces_equal_mirror_pair_flux(tau_mode):
    mi, Q, cfg, m, dt, tot, totd, scale = _setup(tau_mode)
    exp, expd = _wall_totals(m, Q, cfg, dt, "mirror")
    assert np.abs(tot - exp).max() <= 1e-13 * scale.max(), (tot, exp)
    assert np.abs(totd - expd).max() <= 1e-13 * max(1.0, np.abs(expd).max()), (totd, expd)
