"""Oracle pins: least squares (O4), smoothness indicators and WENO (O5/O6).

Independent checks: cell averages of polynomials from closed-form simplex
moments; beta from a Duffy quadrature of its definition; the
collapse of Eq. (weno) when all beta are equal."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W


def tet_means(mi):
    """mean of 1, x, x x^T over each tet, from vertex sums (independent of the oracle)."""
    v = mi.xyz[mi.cell_nodes[:, :4]]
    s = v.sum(1)
    c = s / 4
    xxT = (np.einsum("nka,nkb->nab", v, v) + np.einsum("na,nb->nab", s, s)) / 20.0
    return c, xxT


def poly_means(mi, lin, quad, const=0.0):
    """cell means of const + lin.x + x^T quad x on tets."""
    c, xxT = tet_means(mi)
    return const + c @ lin + np.einsum("nab,ab->n", xxT, quad)


def interior_cells(m, mi, margin):
    V, c, _ = m.geometry()
    L = mi.periodic_length
    ok = []
    for i in range(m.n_cells):
        ids, sh = m.big_stencil(i)
        if np.abs(sh).max() == 0 and np.all(c[i] > margin) and np.all(c[i] < L - margin):
            ok.append(i)
    return ok


@pytest.mark.parametrize("jit", [0.0, 0.12])
def test_linear_field_reproduced_by_every_polynomial(jit):
    """linear data -> every P_m reproduces the gradient (<= 1e-10)."""
    mi = W.kuhn_box(8, jitter=jit)
    m = O.OracleMesh(mi)
    g = np.array([1.0, 2.0, 3.0])
    q = poly_means(mi, g, np.zeros((3, 3)), 5.0)
    Q = np.stack([q, 2 * q, -q, 0.5 * q, q + 10], axis=1)
    for i in interior_cells(m, mi, 0.6)[:20]:
        fit = m.fit_cell(Q, i)
        a, b = fit["a"], fit["b"]
        for v, s in enumerate([1, 2, -1, 0.5, 1]):
            assert np.allclose(a[:3, v], s * g, atol=1e-10 * 3)
            assert np.abs(a[3:, v]).max() < 1e-9
            for mm in range(b.shape[0]):
                assert np.allclose(b[mm, :, v], s * g, atol=1e-10 * 3)
        # equal betas -> linear weights -> WENO value = the linear function (A.6)
        assert np.allclose(fit["wbar"][0], 0.9) and np.allclose(fit["wbar"][1:], 0.025)
        V, c, _ = m.geometry()
        x = c[i] + np.array([[0.03, -0.02, 0.01], [0.0, 0.05, -0.04]])
        val, grad = m.weno_points(Q, i, x)
        exact = 5.0 + x @ g
        assert np.allclose(val[:, 0], exact, atol=1e-12)
        assert np.allclose(grad[:, 0], g, atol=1e-10)


def test_quadratic_field_reproduced_by_p0():
    """x^2 averages -> P_0 has a_xx = 1, other quadratic coefficients 0."""
    mi = W.kuhn_box(8, jitter=0.1)
    m = O.OracleMesh(mi)
    quad = np.zeros((3, 3))
    quad[0, 0] = 1.0
    quad[1, 2] = quad[2, 1] = 0.5   # + y z
    q = poly_means(mi, np.zeros(3), quad, 1.0)
    Q = np.repeat(q[:, None], 5, axis=1)
    V, c, _ = m.geometry()
    for i in interior_cells(m, mi, 0.6)[:10]:
        a = m.fit_cell(Q, i)["a"][:, 0]
        # basis centred at c_i: x^2 + yz = X^2 + 2 c_x X + Y Z + c_z Y + c_y Z + const
        cx, cy, cz = c[i]
        expect = np.array([2 * cx, cz, cy, 1.0, 0.0, 0.0, 0.0, 0.0, 1.0])
        assert np.allclose(a, expect, atol=1e-9), (a, expect)


def test_linear_weight_gradients_exact_for_quadratics():
    """Reading R9s (dq0_mode 2): Eq. (weno) with gamma in place of omega-bar collapses to P_0
    (SURVEY A.6), so on quadratic data its gradient is the exact gradient at any point,
    while the nonlinear weights (power 1) mix in the sub-stencil slopes."""
    mi = W.kuhn_box(8, jitter=0.1)
    m = O.OracleMesh(mi)
    lin = np.array([0.3, -0.2, 0.1])
    quad = np.array([[0.5, 0.1, 0.0], [0.1, -0.3, 0.2], [0.0, 0.2, 0.4]])
    q = poly_means(mi, lin, quad, 2.0)
    Q = np.repeat(q[:, None], 5, axis=1)
    V, c, _ = m.geometry()
    rng = np.random.default_rng(3)
    worst_nl = 0.0
    for i in interior_cells(m, mi, 0.6)[:8]:
        x = c[i] + rng.uniform(-0.1, 0.1, size=(4, 3))
        exact = lin[None, :] + 2 * x @ quad
        _, g_lin = m.weno_points(Q, i, x, linear=True)
        _, g_nl = m.weno_points(Q, i, x)
        assert np.abs(g_lin[:, 0] - exact).max() <= 1e-10
        worst_nl = max(worst_nl, np.abs(g_nl[:, 0] - exact).max())
    assert worst_nl > 1e-6


def test_constant_field_zero_coefficients():
    mi = W.kuhn_box(5)
    m = O.OracleMesh(mi)
    Q = np.tile([1.3, 0.2, -0.1, 0.4, 3.0], (mi.n_cells, 1))
    fit = m.fit_cell(Q, 17)
    assert np.abs(fit["a"]).max() < 1e-13 and np.abs(fit["b"]).max() < 1e-13
    assert np.abs(fit["beta"]).max() < 1e-20
    assert np.allclose(fit["wbar"].sum(0), 1.0)


def test_beta_unit_cube_linear():
    """P = x on a unit cube cell -> beta = 1 (all stencils)."""
    mi = W.cartesian_hex_box(6, h=1.0)
    m = O.OracleMesh(mi)
    V, c, _ = m.geometry()
    i = (2 * 6 + 2) * 6 + 2   # cube (2,2,2): its stencil does not wrap
    ids, sh = m.big_stencil(i)
    assert np.abs(sh).max() == 0
    q = c[:, 0][: m.n_cells]  # cell means of x on unit cubes
    Q = np.stack([q + 2, q * 0 + 1, q * 0, q * 0, q * 0 + 5], 1)
    fit = m.fit_cell(Q, i)
    assert np.allclose(fit["beta"][:, 0], 1.0, atol=1e-12)


def duffy(order=8):
    g, w = np.polynomial.legendre.leggauss(order)
    g = 0.5 * (g + 1)
    w = 0.5 * w
    P, Wt = [], []
    for a, wa in zip(g, w):
        for b, wb in zip(g, w):
            for cc, wc in zip(g, w):
                P.append((a * (1 - b) * (1 - cc), b * (1 - cc), cc))
                Wt.append(wa * wb * wc * (1 - b) * (1 - cc) ** 2)
    return np.array(P), np.array(Wt)


def test_beta_definition_by_quadrature():
    """beta_0 = sum_{|l|=1,2} V^{2|l|/3-1} int (d^l P0)^2 (R15) by brute-force quadrature."""
    mi = W.kuhn_box(6, jitter=0.1)
    m = O.OracleMesh(mi)
    rng = np.random.default_rng(5)
    Q = 1.0 + 0.1 * rng.standard_normal((mi.n_cells, 5))
    Vs, c, M2 = m.geometry()
    P, Wt = duffy()
    for i in [3, 77, 400]:
        fit = m.fit_cell(Q, i)
        v = mi.xyz[mi.cell_nodes[i, :4]]
        X = v[0] + P @ (v[1:] - v[0])          # quadrature points
        V = abs(np.linalg.det(v[1:] - v[0])) / 6
        wts = Wt * 6 * V                      # sum = V
        Xc = X - c[i]
        for comp in range(5):
            a = fit["a"][:, comp]
            gx = a[0] + 2 * a[3] * Xc[:, 0] + a[6] * Xc[:, 1] + a[7] * Xc[:, 2]
            gy = a[1] + 2 * a[4] * Xc[:, 1] + a[6] * Xc[:, 0] + a[8] * Xc[:, 2]
            gz = a[2] + 2 * a[5] * Xc[:, 2] + a[7] * Xc[:, 0] + a[8] * Xc[:, 1]
            b1 = V ** (-1 / 3) * (wts * (gx ** 2 + gy ** 2 + gz ** 2)).sum()
            sec = [2 * a[3], 2 * a[4], 2 * a[5], a[6], a[7], a[8]]
            b2 = V ** (1 / 3) * V * sum(s * s for s in sec)
            assert abs(fit["beta"][0, comp] - (b1 + b2)) <= 1e-11 * (b1 + b2)
            for mm in range(4):
                b = fit["b"][mm, :, comp]
                assert abs(fit["beta"][1 + mm, comp] - V ** (2 / 3) * (b @ b)) <= 1e-12 * V ** (2 / 3) * (b @ b) + 1e-300


def test_weights_sum_to_one_and_eq_weno_literal():
    """Sum of normalised weights is 1 and the point value is Eq. (weno)."""
    mi = W.kuhn_box(6)
    m = O.OracleMesh(mi)
    Q = W.density_step_ic(mi)
    V, c, M2 = m.geometry()
    i = 200
    fit = m.fit_cell(Q, i)
    wbar, beta = fit["wbar"], fit["beta"]
    assert np.allclose(wbar.sum(0), 1.0, atol=1e-15)
    # recompute the weights from the betas (printed formula, power 1, eps 1e-10)
    M = 4
    tz = np.abs(beta[0] - beta[1:]).sum(0) / M
    gam = np.array([1 - 0.025 * M] + [0.025] * M)[:, None]
    w = gam * (1 + tz / (beta + 1e-10))
    assert np.allclose(wbar, w / w.sum(0), rtol=1e-13)
    x = c[i] + np.array([0.05, 0.02, -0.03])
    val, grad = m.weno_points(Q, i, x)
    X = x - c[i]
    a, b = fit["a"], fit["b"]
    mono = np.array([X[0], X[1], X[2], X[0] ** 2 - M2[i, 0, 0], X[1] ** 2 - M2[i, 1, 1], X[2] ** 2 - M2[i, 2, 2],
                     X[0] * X[1] - M2[i, 0, 1], X[0] * X[2] - M2[i, 0, 2], X[1] * X[2] - M2[i, 1, 2]])
    P0 = Q[i] + mono @ a
    Pm = Q[i][None, :] + np.einsum("a,mav->mv", X, b)
    g0 = 1 - 0.025 * M
    expect = wbar[0] * (P0 / g0 - (0.025 / g0) * Pm.sum(0)) + (wbar[1:] * Pm).sum(0)
    assert np.allclose(val[0], expect, rtol=1e-14, atol=1e-14)
