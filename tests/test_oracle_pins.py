"""Oracle pins added in round 2 for the parts round 1 left unpinned (VERDICT r01 "weak" 2):
the time step (R6), the tet sub-stencil member lists (R16), the nonlinear WENO weights
(R13-R15) at hand-computed smoothness indicators, and the positivity
fallback (R21) on a state where it fires.  Each expected value below comes from the
paper / SPEC worked examples, from closed forms worked by hand, or from brute force
independent of the oracle's code; none is read back from the oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W

GAMMA = 1.4


# --------------------------------------------------------------------------- #
# R6 time step
# --------------------------------------------------------------------------- #
def test_dt_spec_worked_example():
    """uniform rho = 1, p = 1/gamma, U = 0, inviscid, unit-cube cells,
    CFL 0.5 -> c = 1, h = V / max face area = 1, dt = 0.5."""
    mi = W.cartesian_hex_box(5, h=1.0)
    Q = W.uniform_state(mi.n_cells, 1.0, (0.0, 0.0, 0.0), 1.0 / GAMMA)
    s = O.OracleSolver(O.OracleMesh(mi), Q, O.OracleConfig(cfl=0.5))
    assert abs(s.dt() - 0.5) <= 1e-15


def test_dt_halves_with_cell_size_and_viscous_closed_form():
    """S:341 'halving every cell size halves dt (inviscid)'; and with nu: on unit cubes,
    rho = 1, p = 1/gamma (T = 1/gamma = T_inf, so mu = mu_inf), |U| = 0.6, mu = 0.1:
    dt = 0.5 * 1 / (0.6 + 1 + 2 * 0.1 / 1) = 0.5 / 1.8."""
    vel = (0.6, 0.0, 0.0)
    d = []
    for h in (1.0, 0.5):
        mi = W.cartesian_hex_box(5, h=h)
        Q = W.uniform_state(mi.n_cells, 1.0, vel, 1.0 / GAMMA)
        d.append(O.OracleSolver(O.OracleMesh(mi), Q, O.OracleConfig(cfl=0.5)).dt())
    assert abs(d[1] / d[0] - 0.5) <= 1e-14
    assert abs(d[0] - 0.5 / 1.6) <= 1e-15
    mi = W.cartesian_hex_box(5, h=1.0)
    Q = W.uniform_state(mi.n_cells, 1.0, vel, 1.0 / GAMMA)
    cfg = O.OracleConfig(cfl=0.5, tau_mode=1, mu_inf=0.1, t_inf=1.0 / GAMMA)
    assert abs(O.OracleSolver(O.OracleMesh(mi), Q, cfg).dt() - 0.5 / 1.8) <= 1e-15


def test_dt_on_jittered_tets_uses_volume_over_largest_face():
    """R6 on unstructured tets: h_i = V_i / max_p S_ip from independently computed
    determinants and cross products; one cell made fast so the minimum is known."""
    mi = W.kuhn_box(5, jitter=0.1)
    v = mi.xyz[mi.cell_nodes[:, :4]]
    V = np.abs(np.einsum("ij,ij->i", v[:, 1] - v[:, 0], np.cross(v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]))) / 6.0
    area = np.stack([0.5 * np.linalg.norm(np.cross(v[:, b] - v[:, a], v[:, c] - v[:, a]), axis=1)
                     for (a, b, c) in ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))], axis=1)
    h = V / area.max(axis=1)
    Q = W.uniform_state(mi.n_cells, 1.0, (0.0, 0.0, 0.0), 1.0 / GAMMA)  # c = 1 everywhere
    assert abs(O.OracleSolver(O.OracleMesh(mi), Q, O.OracleConfig(cfl=0.3)).dt() - 0.3 * h.min()) <= 1e-15
    # a cell moving at |U| = 9 (c = 1 there): dt = 0.3 h_k / 10 if that is the minimum
    k = int(np.argmax(h))
    Q[k, 1] = 9.0
    Q[k, 4] += 0.5 * 81.0
    exp = 0.3 * min(h[k] / 10.0, np.delete(h, k).min())
    assert abs(O.OracleSolver(O.OracleMesh(mi), Q, O.OracleConfig(cfl=0.3)).dt() - exp) <= 1e-15


# --------------------------------------------------------------------------- #
# R16 tet sub-stencils
# --------------------------------------------------------------------------- #
def ordered_tet_neighbours(mi, N):
    """nb[c][p] = the cell across the face opposite local node p of cell c, from node keys
    of the periodic Kuhn box (independent of the oracle's connectivity)."""
    ijk = np.rint(mi.xyz / (2.0 / N)).astype(int) % N
    wrapped = ijk[:, 0] * N * N + ijk[:, 1] * N + ijk[:, 2]
    owners = {}
    for c in range(mi.n_cells):
        nodes = wrapped[mi.cell_nodes[c, :4]]
        for p in range(4):
            owners.setdefault(tuple(sorted(np.delete(nodes, p))), []).append((c, p))
    nb = np.full((mi.n_cells, 4), -1, np.int64)
    for key, cp in owners.items():
        assert len(cp) == 2
        (a, pa), (b, pb) = cp
        nb[a, pa] = b
        nb[b, pb] = a
    return nb


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_tet_substencil_members_R16(jitter):
    """S_{i_1} = {i_1, i_2, i_3, i_11, i_12, i_13}, S_{i_2} = {i_1, i_2, i_4, i_2*},
    S_{i_3} = {i_2, i_3, i_4, i_3*}, S_{i_4} = {i_3, i_1, i_4, i_4*} (target
    cell i implied), where i_m* are i_m's face neighbours other than i in i_m's face
    order (R16); member lists compared in order."""
    N = 5
    mi = W.kuhn_box(N, jitter=jitter)
    nb = ordered_tet_neighbours(mi, N)
    m = O.OracleMesh(mi)
    triples = [(0, 1, 2), (0, 1, 3), (1, 2, 3), (2, 0, 3)]
    for i in range(m.n_cells):
        ids, _ = m.big_stencil(i)
        assert list(ids[:4]) == list(nb[i])  # first layer in face order
        for mm in range(4):
            im = nb[i, mm]
            exp = [nb[i, t] for t in triples[mm]] + [x for x in nb[im] if x != i]
            seen = []
            for x in exp:  # de-duplicated (none on Kuhn meshes)
                if x != i and x not in seen:
                    seen.append(x)
            assert list(m.sub_stencil(i, mm)) == seen, (i, mm)


# --------------------------------------------------------------------------- #
# nonlinear weights at hand-computed smoothness indicators
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("omega_pow", [1, 2])
def test_weno_weights_hand_values(omega_pow):
    """Unit-cube hexes, density cell averages of rho = 2 + (z - z_i)^2 around an interior
    cell i (every other variable uniform).  By hand:
      P_0 is the exact quadratic (z - z_i)^2 - 1/12, so beta_0 = |Omega|^{-1/3} int (2z)^2
        + |Omega|^{1/3} int 2^2 = 1/3 + 4 = 13/3;
      every hex sub-stencil {i, i_1 or i_6, two ring cells} interpolates exactly: slopes
        (0, 0, -1) or (0, 0, +1), so beta_m = 1 (m = 1..8);
      tau_Z = sum_m |beta_0 - beta_m| / M = 10/3;
      omega_0 = 0.8 (1 + r_0^p), r_0 = (10/3)/(13/3 + eps); omega_m = 0.025 (1 + r^p),
      r = (10/3)/(1 + eps), eps = 1e-10 (R14)."""
    mi = W.cartesian_hex_box(7, h=1.0)
    c = mi.xyz[mi.cell_nodes].mean(axis=1)
    i = int(np.argmin(np.abs(c - 3.5).sum(axis=1)))
    k = np.rint(c[:, 2] - c[i, 2])
    Q = W.uniform_state(mi.n_cells, 1.0, (0.0, 0.0, 0.0), 1.0)  # momentum 0, rhoE uniform
    Q[:, 0] = 2.0 + k * k + 1.0 / 12.0
    m = O.OracleMesh(mi)
    r = m.fit_cell(Q, i, O.OracleConfig(omega_pow=omega_pow))
    beta, wbar = r["beta"][:, 0], r["wbar"][:, 0]
    assert abs(beta[0] - 13.0 / 3.0) <= 1e-12 and np.abs(beta[1:] - 1.0).max() <= 1e-12, beta
    eps = 1e-10
    w0 = 0.8 * (1 + ((10.0 / 3.0) / (13.0 / 3.0 + eps)) ** omega_pow)
    wm = 0.025 * (1 + ((10.0 / 3.0) / (1.0 + eps)) ** omega_pow)
    tot = w0 + 8 * wm
    assert abs(wbar[0] - w0 / tot) <= 1e-13 and np.abs(wbar[1:] - wm / tot).max() <= 1e-13, wbar
    # the uniform variables have beta = 0 everywhere: linear weights (tau_Z = 0)
    for v in range(1, 5):
        assert np.abs(r["wbar"][:, v] - np.array([0.8] + [0.025] * 8)).max() <= 1e-15


# --------------------------------------------------------------------------- #
# R21 positivity fallback
# --------------------------------------------------------------------------- #
def test_positivity_fallback_count_is_brute_force_count():
    """After one step of the spike state some reconstructed Gauss-point states are not
    admissible: the residual's fallback count equals the number of (face, Gauss point,
    side) reconstructions with rho <= 0 or p <= 0, found by evaluating each side's
    polynomial at every Gauss point and testing it here; mass stays conserved."""
    mi = W.kuhn_box(6)
    m = O.OracleMesh(mi)
    s = O.OracleSolver(m, W.spike_state(mi), O.OracleConfig(cfl=0.3))
    s.step(1)
    Q1, t, dt, fb_step = s.state()
    L, dL, fb = s.residual(Q1, dt)
    f = m.faces()
    bad = 0
    for fi in range(m.n_faces):
        ng = f["ngp"][fi]
        x = f["gp_x"][fi, :ng]
        for cell, xs in ((f["owner"][fi], x), (f["nb"][fi], x - f["shift"][fi])):
            val, _ = m.weno_points(Q1, int(cell), xs)
            p = (GAMMA - 1.0) * (val[:, 4] - 0.5 * (val[:, 1:4] ** 2).sum(1) / val[:, 0])
            bad += int(np.sum((val[:, 0] <= 0) | (p <= 0)))
    assert bad > 0 and fb == bad, (fb, bad)
    V = m.geometry()[0][: m.n_cells]
    assert abs((L[:, 0] * V).sum()) <= 1e-12 * np.abs(L[:, 0] * V).max()
