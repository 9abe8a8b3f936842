"""Oracle pins: Maxwellian moments, micro-slopes and the Gauss-point GKS flux.

The independent side integrates over velocity space NUMERICALLY (Gauss-Legendre
split at u = 0; radial quadrature for the K = 2 internal degrees of freedom)
and over time numerically, evaluating Eq. (flux) term by term, and
checks the tau = 0 result against the Euler-chain identity with analytic
Euler Jacobians, which shares nothing with the kinetic code.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W

GAMMA = 1.4
K = (5 - 3 * GAMMA) / (GAMMA - 1)  # = 2


# --------------------------------------------------------------------------- #
# numerical velocity-space machinery (independent of the oracle)
# --------------------------------------------------------------------------- #
def gl(a, b, n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (b - a) * x + 0.5 * (a + b), 0.5 * (b - a) * w


def moments_1d(U, lam, rng="full", nmax=9, n=80):
    """<u^k> of sqrt(lam/pi) exp(-lam (u-U)^2) over the full line or a half line."""
    s = 1.0 / np.sqrt(lam)
    lo, hi = U - 14 * s, U + 14 * s
    pieces = []
    if rng == "full":
        if lo < 0 < hi:
            pieces = [(lo, 0.0), (0.0, hi)]
        else:
            pieces = [(lo, hi)]
    elif rng == "pos":
        if hi > 0:
            pieces = [(max(lo, 0.0), hi)]
    else:
        if lo < 0:
            pieces = [(lo, min(hi, 0.0))]
    out = np.zeros(nmax + 1)
    for a, b in pieces:
        # split further for accuracy
        for a2, b2 in zip(np.linspace(a, b, 9)[:-1], np.linspace(a, b, 9)[1:]):
            x, w = gl(a2, b2, n)
            f = np.sqrt(lam / np.pi) * np.exp(-lam * (x - U) ** 2)
            out += np.array([(w * f * x ** k).sum() for k in range(nmax + 1)])
    return out


def xi_moments(lam, dmax=4):
    """<(xi^2)^d> for K = 2 internal degrees of freedom, by radial quadrature."""
    s = 1.0 / np.sqrt(lam)
    r, w = gl(0.0, 14 * s, 200)
    f = (lam / np.pi) * np.exp(-lam * r * r) * 2 * np.pi * r
    return np.array([(w * f * r ** (2 * d)).sum() for d in range(dmax + 1)])


class Table:
    def __init__(self, rho, U, V, Wv, lam, rng):
        self.rho = rho
        self.u = moments_1d(U, lam, rng)
        self.v = moments_1d(V, lam, "full")
        self.w = moments_1d(Wv, lam, "full")
        self.x = xi_moments(lam)

    def mom(self, P):
        """P: dict (a,b,c,d) -> coefficient, polynomial in u, v, w, xi^2."""
        return sum(c * self.u[a] * self.v[b] * self.w[cc] * self.x[d] for (a, b, cc, d), c in P.items())


def pmul(P, Q):
    R = {}
    for (a, b, c, d), x in P.items():
        for (e, f, g, h), y in Q.items():
            k = (a + e, b + f, c + g, d + h)
            R[k] = R.get(k, 0.0) + x * y
    return R


def padd(*Ps):
    R = {}
    for P in Ps:
        for k, v in P.items():
            R[k] = R.get(k, 0.0) + v
    return R


def pscale(P, s):
    return {k: v * s for k, v in P.items()}


PSI = [{(0, 0, 0, 0): 1.0}, {(1, 0, 0, 0): 1.0}, {(0, 1, 0, 0): 1.0}, {(0, 0, 1, 0): 1.0},
       {(2, 0, 0, 0): 0.5, (0, 2, 0, 0): 0.5, (0, 0, 2, 0): 0.5, (0, 0, 0, 1): 0.5}]
UVEC = [{(1, 0, 0, 0): 1.0}, {(0, 1, 0, 0): 1.0}, {(0, 0, 1, 0): 1.0}]


def prim(q):
    rho = q[0]
    U, V, Wv = q[1] / rho, q[2] / rho, q[3] / rho
    lam = (K + 3) * rho / (4 * (q[4] - 0.5 * rho * (U * U + V * V + Wv * Wv)))
    return rho, U, V, Wv, lam


def slope_poly(a):
    return padd(*[pscale(PSI[j], a[j]) for j in range(5)])


def solve_slope(T_full, b):
    M = np.array([[T_full.mom(pmul(PSI[i], PSI[j])) for j in range(5)] for i in range(5)])
    return np.linalg.solve(M, np.asarray(b) / T_full.rho)


def slopes(q, dq):
    rho, U, V, Wv, lam = prim(q)
    T = Table(rho, U, V, Wv, lam, "full")
    a = [solve_slope(T, dq[j]) for j in range(3)]
    au = padd(*[pmul(slope_poly(a[j]), UVEC[j]) for j in range(3)])
    b = [-rho * T.mom(pmul(au, PSI[i])) for i in range(5)]
    A = solve_slope(T, b)
    return a, A, au


def kinetic_dq0(ql, dql, qr, dqr):
    """Reading R9k by numerical quadrature: d_j Q0 = rho_l <a^l_j psi>_{u>0} + rho_r <a^r_j psi>_{u<0},
    the j-derivative of Q0 = int_{u>0} psi g_l + int_{u<0} psi g_r with d_j g_k = a^k_j g_k."""
    rl, Ul, Vl, Wl, laml = prim(ql)
    rr, Ur, Vr, Wr, lamr = prim(qr)
    Tl_pos = Table(rl, Ul, Vl, Wl, laml, "pos")
    Tr_neg = Table(rr, Ur, Vr, Wr, lamr, "neg")
    al, _, _ = slopes(ql, dql)
    ar, _, _ = slopes(qr, dqr)
    return np.array([[rl * Tl_pos.mom(pmul(slope_poly(al[j]), PSI[i])) + rr * Tr_neg.mom(pmul(slope_poly(ar[j]), PSI[i]))
                      for i in range(5)] for j in range(3)])


def brute_force_flux(ql, dql, qr, dqr, tau, delta, nt=24, dq0_mode=0):
    """Numerical int_0^delta int psi u f dXi dt of Eq. (flux), local frame."""
    rl, Ul, Vl, Wl, laml = prim(ql)
    rr, Ur, Vr, Wr, lamr = prim(qr)
    Tl_pos = Table(rl, Ul, Vl, Wl, laml, "pos")
    Tr_neg = Table(rr, Ur, Vr, Wr, lamr, "neg")
    Q0 = np.array([rl * Tl_pos.mom(PSI[i]) + rr * Tr_neg.mom(PSI[i]) for i in range(5)])
    r0, U0, V0, W0, lam0 = prim(Q0)
    T0 = Table(r0, U0, V0, W0, lam0, "full")
    if dq0_mode == 0:
        dq0 = 0.5 * (np.asarray(dql) + np.asarray(dqr))  # reading R9
    else:
        dq0 = kinetic_dq0(ql, dql, qr, dqr)  # reading R9k
    a0, A0, au0 = slopes(Q0, dq0)
    al, Al, aul = slopes(ql, dql)
    ar, Ar, aur = slopes(qr, dqr)
    U = UVEC[0]
    t, wt = gl(0.0, delta, nt)
    I = np.zeros(5)
    for tk, wk in zip(t, wt):
        e = np.exp(-tk / tau) if tau > 0 else 0.0
        for i in range(5):
            upsi = pmul(U, PSI[i])
            F = r0 * ((1 - e) * T0.mom(upsi) + ((tk + tau) * e - tau) * T0.mom(pmul(au0, upsi))
                      + (tk - tau + tau * e) * T0.mom(pmul(slope_poly(A0), upsi)))
            F += rr * e * (Tr_neg.mom(upsi) - (tau + tk) * Tr_neg.mom(pmul(aur, upsi))
                           - tau * Tr_neg.mom(pmul(slope_poly(Ar), upsi)))
            F += rl * e * (Tl_pos.mom(upsi) - (tau + tk) * Tl_pos.mom(pmul(aul, upsi))
                           - tau * Tl_pos.mom(pmul(slope_poly(Al), upsi)))
            I[i] += wk * F
    return I, Q0


def random_gp(rng):
    rho, vel, p = W.random_states(2, seed=int(rng.integers(1 << 30)))
    qs = []
    for k in range(2):
        q = np.array([rho[k], *(rho[k] * vel[k] * 0.3), p[k] / (GAMMA - 1) + 0.5 * rho[k] * (vel[k] * 0.3) @ (vel[k] * 0.3)])
        dq = rng.normal(size=(3, 5)) * 0.3 * np.abs(q)[None, :]
        qs += [q, dq]
    return qs


# --------------------------------------------------------------------------- #
def test_moments_vs_quadrature():
    """full and half-range moments vs numerical quadrature."""
    rng = np.random.default_rng(20240700)
    for _ in range(30):
        U = rng.uniform(-3, 3)
        lam = rng.uniform(0.05, 5)
        for name in ("full", "pos", "neg"):
            u, v, w, xi = O.moments([1.0, U, 0.3, -0.2, lam], K, name)
            ref = moments_1d(U, lam, name, nmax=7)
            # tolerance per order relative to the full-line moment of |u|^k: the
            # half-range recursion is accurate relative to that scale (tails lose
            # relative digits, as for any upward recursion)
            scale = moments_1d(abs(U), lam, "full", nmax=7) + (abs(U) + 1 / np.sqrt(lam)) ** np.arange(8)
            assert np.all(np.abs(u - ref) <= 1e-12 * scale), (u - ref) / scale
        up, _, _, _ = O.moments([1.0, U, 0, 0, lam], K, "pos")
        un, _, _, _ = O.moments([1.0, U, 0, 0, lam], K, "neg")
        uf, _, _, xi = O.moments([1.0, U, 0, 0, lam], K, "full")
        assert np.allclose(up + un, uf, rtol=1e-13, atol=1e-13)
        assert np.allclose(xi[:3], xi_moments(lam)[:3], rtol=1e-12)
    # SPEC example: rho=1, U=0, lambda=1 -> <u>_{>0} = 1/(2 sqrt(pi))
    up, _, _, _ = O.moments([1.0, 0.0, 0.0, 0.0, 1.0], K, "pos")
    assert abs(up[1] - 0.5 / np.sqrt(np.pi)) < 1e-15 and abs(up[2] - 0.25) < 1e-15


def test_micro_slope_vs_numerical_solve():
    rng = np.random.default_rng(1)
    for _ in range(10):
        q, dq, _, _ = random_gp(rng)
        b = dq[0]
        a = O.micro_slope(q, K, b)
        rho, U, V, Wv, lam = prim(q)
        ref = solve_slope(Table(rho, U, V, Wv, lam, "full"), b)
        assert np.allclose(a, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
        # round trip: rho <a psi_i> = b_i
        T = Table(rho, U, V, Wv, lam, "full")
        back = [rho * T.mom(pmul(slope_poly(a), PSI[i])) for i in range(5)]
        assert np.allclose(back, b, rtol=1e-10, atol=1e-12 * np.abs(b).max())
    assert np.allclose(O.micro_slope(q, K, np.zeros(5)), 0.0)


@pytest.mark.parametrize("tau,delta", [(0.07, 0.05), (0.07, 0.1), (0.0, 0.08), (0.01, 0.2)])
def test_gp_flux_vs_brute_force(tau, delta):
    """Eq. (flux) integrated literally over velocity and time."""
    rng = np.random.default_rng(int(1000 * (tau + delta)))
    cfg = O.OracleConfig(tau_mode=1 if tau > 0 else 0)
    for _ in range(3):
        ql, dql, qr, dqr = random_gp(rng)
        if tau > 0:
            # choose mu so that tau = mu/p0 exactly (c1 = 0): need p0 first
            o = O.gp_flux(ql, dql, qr, dqr, 2 * delta, O.OracleConfig())
            r0, U0, V0, W0, lam0 = prim(o["Q0"])
            p0 = r0 / (2 * lam0)
            cfg = O.OracleConfig(tau_mode=1, c1=0.0, mu_inf=tau * p0, t_inf=p0 / r0, mu_exp=0.7)
        o = O.gp_flux(ql, dql, qr, dqr, 2 * delta, cfg)
        assert abs(o["tau"] - tau) < 1e-14
        I_half, Q0 = brute_force_flux(ql, dql, qr, dqr, tau, delta)
        I_full, _ = brute_force_flux(ql, dql, qr, dqr, tau, 2 * delta)
        assert np.allclose(o["Q0"], Q0, rtol=1e-12)
        scale = np.abs(I_full).max()
        assert np.abs(o["I_half"] - I_half).max() <= 1e-10 * scale
        assert np.abs(o["I_full"] - I_full).max() <= 1e-10 * scale


@pytest.mark.parametrize("tau,delta", [(0.07, 0.1), (0.0, 0.08)])
def test_gp_flux_kinetic_dq0_vs_brute_force(tau, delta):
    """Reading R9k (dq0_mode 1): the equilibrium slopes are the numerically integrated
    half-range moments of the side slopes, and the whole Gauss-point flux matches the literal
    velocity/time quadrature of Eq. (flux) with them."""
    rng = np.random.default_rng(int(7000 * (tau + delta)))
    for _ in range(3):
        ql, dql, qr, dqr = random_gp(rng)
        cfg = O.OracleConfig(dq0_mode=1)
        if tau > 0:
            o = O.gp_flux(ql, dql, qr, dqr, 2 * delta, O.OracleConfig())
            r0, U0, V0, W0, lam0 = prim(o["Q0"])
            p0 = r0 / (2 * lam0)
            cfg = O.OracleConfig(tau_mode=1, c1=0.0, mu_inf=tau * p0, t_inf=p0 / r0, mu_exp=0.7, dq0_mode=1)
        o = O.gp_flux(ql, dql, qr, dqr, 2 * delta, cfg)
        ref = kinetic_dq0(ql, dql, qr, dqr)
        assert np.abs(o["dq0"] - ref).max() <= 1e-11 * np.abs(ref).max()
        I_half, _ = brute_force_flux(ql, dql, qr, dqr, tau, delta, dq0_mode=1)
        I_full, _ = brute_force_flux(ql, dql, qr, dqr, tau, 2 * delta, dq0_mode=1)
        scale = np.abs(I_full).max()
        assert np.abs(o["I_half"] - I_half).max() <= 1e-10 * scale
        assert np.abs(o["I_full"] - I_full).max() <= 1e-10 * scale
        # R9 (mode 0) is the plain average; the two readings differ for unequal sides
        assert np.allclose(O.gp_flux(ql, dql, qr, dqr, 2 * delta, O.OracleConfig())["dq0"], 0.5 * (dql + dqr),
                           rtol=1e-14, atol=1e-14 * np.abs(dql).max())
        assert np.abs(o["dq0"] - 0.5 * (dql + dqr)).max() > 1e-6 * np.abs(ref).max()


def test_kinetic_dq0_special_cases():
    """R9k limits: equal sides (q_l = q_r, dq_l = dq_r) give dQ0 = dQ (the half-range
    moments add up to the full ones); a strongly supersonic flow to +n (U sqrt(lam) = 12)
    takes dQ0 from the left side alone, and to -n from the right side."""
    rng = np.random.default_rng(5)
    ql, dql, qr, dqr = random_gp(rng)
    o = O.gp_flux(ql, dql, ql, dql, 0.1, O.OracleConfig(dq0_mode=1))
    assert np.abs(o["dq0"] - dql).max() <= 1e-13 * np.abs(dql).max()
    for sgn, side in ((1.0, 0), (-1.0, 1)):
        qa, qb = ql.copy(), qr.copy()
        for q in (qa, qb):
            rho, U, V, Wv, lam = prim(q)
            p = rho / (2 * lam)
            Un = sgn * 12.0 / np.sqrt(lam)
            q[1] = rho * Un
            q[4] = p / (GAMMA - 1) + 0.5 * rho * (Un * Un + V * V + Wv * Wv)
        o = O.gp_flux(qa, dql, qb, dqr, 0.1, O.OracleConfig(dq0_mode=1))
        exp = dql if side == 0 else dqr
        assert np.abs(o["dq0"] - exp).max() <= 1e-9 * np.abs(exp).max()  # moments of |U| ~ 12/sqrt(lam): cancellation


def euler_flux(q):
    rho = q[0]
    u = q[1:4] / rho
    p = (GAMMA - 1) * (q[4] - 0.5 * rho * u @ u)
    return np.array([q[1], q[1] * u[0] + p, q[2] * u[0], q[3] * u[0], u[0] * (q[4] + p)]), p


def euler_jacobian(q, j):
    """Analytic dF_j/dQ of the Euler equations (written out, not differentiated)."""
    g = GAMMA
    rho = q[0]
    u = q[1:4] / rho
    E = q[4] / rho
    q2 = u @ u
    H = g * E - 0.5 * (g - 1) * q2
    A = np.zeros((5, 5))
    e = np.eye(3)[j]
    A[0, 1 + j] = 1.0
    for k in range(3):
        A[1 + k, 0] = -u[k] * u[j] + (g - 1) * 0.5 * q2 * e[k]
        for l in range(3):
            A[1 + k, 1 + l] = u[k] * (1 if l == j else 0) + u[j] * (1 if l == k else 0) - (g - 1) * u[l] * e[k]
        A[1 + k, 4] = (g - 1) * e[k]
    A[4, 0] = u[j] * ((g - 1) * q2 - g * E)
    for l in range(3):
        A[4, 1 + l] = H * (1 if l == j else 0) - (g - 1) * u[l] * u[j]
    A[4, 4] = g * u[j]
    return A


def test_tau0_euler_chain_identity():
    """tau = 0: f = g0 (1 + A t) => F = F_Euler(Q0),
    d_t F = A_n(Q0) (-sum_j A_j(Q0) d_j Q0)."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        ql, dql, qr, dqr = random_gp(rng)
        o = O.gp_flux(ql, dql, qr, dqr, 0.01, O.OracleConfig())
        Q0 = o["Q0"]
        F, _ = euler_flux(Q0)
        d0 = 0.5 * (dql + dqr)
        dtQ = -sum(euler_jacobian(Q0, j) @ d0[j] for j in range(3))
        dF = euler_jacobian(Q0, 0) @ dtQ
        assert np.allclose(o["F"], F, rtol=1e-12, atol=1e-12 * np.abs(F).max())
        assert np.allclose(o["dF"], dF, rtol=1e-9, atol=1e-11 * np.abs(dF).max())


def test_uniform_state_is_euler_flux_any_tau():
    """g_l = g_r = g0 and zero slopes -> Euler flux for any tau."""
    rho, vel, p = W.random_states(5, seed=3)
    for k in range(5):
        q = np.array([rho[k], *(rho[k] * vel[k]), p[k] / (GAMMA - 1) + 0.5 * rho[k] * vel[k] @ vel[k]])
        z = np.zeros((3, 5))
        F, _ = euler_flux(q)
        for cfg in (O.OracleConfig(), O.OracleConfig(tau_mode=1, mu_inf=0.3, c1=0.0)):
            o = O.gp_flux(q, z, q, z, 0.02, cfg)
            assert np.allclose(o["I_full"], 0.02 * F, rtol=1e-12, atol=1e-13 * np.abs(F).max())
            assert np.allclose(o["F"], F, rtol=1e-11, atol=1e-12 * np.abs(F).max())
            assert np.allclose(o["dF"], 0.0, atol=1e-9 * np.abs(F).max())
            assert np.allclose(o["Q0"], q, rtol=1e-13)


def test_collisionless_limit_is_kfvs():
    """tau -> infinity with zero slopes -> kinetic flux-vector splitting."""
    ql = np.array([1.0, 0.3, 0.1, 0.0, 2.6])
    qr = np.array([0.5, -0.1, 0.0, 0.2, 1.4])
    z = np.zeros((3, 5))
    cfg = O.OracleConfig(tau_mode=1, mu_inf=1e4, c1=0.0)
    d = 1e-3
    o = O.gp_flux(ql, z, qr, z, 2 * d, cfg)
    rl, Ul, Vl, Wl, laml = prim(ql)
    rr, Ur, Vr, Wr, lamr = prim(qr)
    Tl, Tr = Table(rl, Ul, Vl, Wl, laml, "pos"), Table(rr, Ur, Vr, Wr, lamr, "neg")
    kfvs = np.array([rl * Tl.mom(pmul(UVEC[0], PSI[i])) + rr * Tr.mom(pmul(UVEC[0], PSI[i])) for i in range(5)])
    assert np.allclose(o["I_full"] / (2 * d), kfvs, rtol=1e-5)


def test_time_fit_round_trip():
    """the fitted F, dF reproduce both sub-interval integrals."""
    rng = np.random.default_rng(11)
    ql, dql, qr, dqr = random_gp(rng)
    dt = 0.03
    o = O.gp_flux(ql, dql, qr, dqr, dt, O.OracleConfig(tau_mode=1, mu_inf=0.01))
    s = np.abs(o["I_full"]).max()
    assert np.allclose(o["F"] * dt + 0.5 * o["dF"] * dt ** 2, o["I_full"], atol=1e-14 * s)
    assert np.allclose(0.5 * o["F"] * dt + 0.125 * o["dF"] * dt ** 2, o["I_half"], atol=1e-14 * s)


def test_local_frame_orthonormal():
    rng = np.random.default_rng(2)
    for _ in range(50):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        t1, t2 = O.local_frame(n)
        R = np.stack([n, t1, t2])
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-15)
        assert abs(np.linalg.det(R) - 1) < 1e-14


def test_farfield_state_consistency():
    """Uniform free stream at a farfield face -> the ghost is the free stream (SPEC S:494 example)."""
    cfg = O.OracleConfig(freestream=(1.0, 0.2535, 0.0, 0.0, 1 / 1.4))
    q = W.uniform_state(1, 1.0, (0.2535, 0, 0), 1 / 1.4)[0]
    for n in (np.array([1.0, 0, 0]), np.array([-1.0, 0, 0]), np.array([0.6, 0.8, 0])):
        assert np.allclose(O.farfield_state(q, n, cfg), q, rtol=1e-13)
    cfg = O.OracleConfig(freestream=(1.0, 1.5, 0.0, 0.0, 1 / 1.4))  # supersonic inflow face
    qi = W.uniform_state(1, 0.8, (0.1, 0, 0), 0.9)[0]
    qf = W.uniform_state(1, 1.0, (1.5, 0, 0), 1 / 1.4)[0]
    assert np.allclose(O.farfield_state(qi, np.array([-1.0, 0, 0]), cfg), qf, rtol=1e-13)


def test_farfield_state_characteristics():
    """Farfield ghost state (R25) against the textbook characteristic boundary
    condition along the face normal, on seeded random states: supersonic outflow
    returns the interior state, supersonic inflow the free stream; subsonic faces
    keep the outgoing invariant R+ = u_n + 2c/(g-1) of the interior and the incoming
    R- = u_n - 2c/(g-1) of the free stream, with tangential velocity and entropy
    p/rho^g from the upwind side."""
    g = 1.4
    rng = np.random.default_rng(20240700)

    def prim(q):
        rho = q[0]; u = q[1:4] / rho
        p = (g - 1) * (q[4] - 0.5 * rho * u @ u)
        return rho, u, p, np.sqrt(g * p / rho)

    seen = set()
    for _ in range(400):
        n = rng.normal(size=3); n /= np.linalg.norm(n)
        rho_i, rho_f = rng.uniform(0.3, 3.0, 2)
        p_i, p_f = rng.uniform(0.3, 3.0, 2)
        ui = rng.normal(size=3) * rng.uniform(0, 2.5)
        uf = rng.normal(size=3) * rng.uniform(0, 2.5)
        qi = np.r_[rho_i, rho_i * ui, p_i / (g - 1) + 0.5 * rho_i * ui @ ui]
        cfg = O.OracleConfig(gamma=g, freestream=(rho_f, *uf, p_f))
        qf = np.r_[rho_f, rho_f * uf, p_f / (g - 1) + 0.5 * rho_f * uf @ uf]
        qb = O.farfield_state(qi, n, cfg)
        _, _, _, c_i = prim(qi)
        _, _, _, c_f = prim(qf)
        un_i, un_f = ui @ n, uf @ n
        rb, ub, pb, cb = prim(qb)
        unb = ub @ n
        if un_i - c_i > 0 and un_f + c_f >= 0:
            seen.add("out")
            assert np.allclose(qb, qi, rtol=1e-12, atol=1e-12)
        elif un_f + c_f < 0 and un_i - c_i <= 0:
            seen.add("in")
            assert np.allclose(qb, qf, rtol=1e-12, atol=1e-12)
        elif abs(un_i) < c_i and abs(un_f) < c_f:
            seen.add("sub")
            assert abs((unb + 2 * cb / (g - 1)) - (un_i + 2 * c_i / (g - 1))) < 1e-11
            assert abs((unb - 2 * cb / (g - 1)) - (un_f - 2 * c_f / (g - 1))) < 1e-11
            up_u, up_rho, up_p = (ui, rho_i, p_i) if unb > 0 else (uf, rho_f, p_f)
            assert np.allclose(ub - unb * n, up_u - (up_u @ n) * n, atol=1e-12)
            assert abs(pb / rb ** g - up_p / up_rho ** g) < 1e-11 * (up_p / up_rho ** g)
    assert seen == {"out", "in", "sub"}, seen


@pytest.mark.parametrize("pr", [0.72, 2.0 / 3.0])
def test_prandtl_heat_flux_ratio(pr):
    """R29 (Prandtl-number fix, energy flux += (1/Pr - 1) x heat flux of the non-equilibrium
    part): a resting gas (rho = p = 1) with a normal temperature gradient at uniform pressure,
    tau << dt (Navier-Stokes regime).  The BGK energy flux is the Chapman-Enskog heat flux
    q = -c_p mu dT/dn with mu = tau p, c_p = gamma/(gamma - 1) (Fourier's law at Pr = 1, a
    textbook result independent of the kinetic code), and with the fix it is q / Pr."""
    g = 0.3                                   # dT/dn; rho = p / T, so d rho/dn = -g at T = 1
    q = np.array([1.0, 0.0, 0.0, 0.0, 1.0 / (GAMMA - 1)])
    dq = np.zeros((3, 5))
    dq[0, 0] = -g
    tau, dt = 1e-6, 1e-3
    base = dict(tau_mode=1, c1=0.0, mu_inf=tau * 1.0, t_inf=1.0, mu_exp=0.7)
    F1 = O.gp_flux(q, dq, q, dq, dt, O.OracleConfig(**base))["F"]
    Fp = O.gp_flux(q, dq, q, dq, dt, O.OracleConfig(prandtl=pr, **base))["F"]
    q_ce = -GAMMA / (GAMMA - 1) * (tau * 1.0) * g
    assert abs(F1[4] / q_ce - 1) < 1e-3, (F1[4], q_ce)
    assert abs(Fp[4] / F1[4] - 1 / pr) < 1e-3, (Fp[4] / F1[4], 1 / pr)
    assert np.allclose(Fp[:4], F1[:4], rtol=0, atol=1e-15)   # only the energy flux changes


def test_prandtl_fix_inactive_without_nonequilibrium():
    """Uniform state (no gradients): f = g0, no heat flux, so Pr changes nothing; tau = 0:
    the non-equilibrium part vanishes identically (R29)."""
    rng = np.random.default_rng(11)
    ql, dql, qr, dqr = random_gp(rng)
    z = np.zeros((3, 5))
    cfg = dict(tau_mode=1, c1=0.0, mu_inf=0.01, t_inf=1.0)
    a = O.gp_flux(ql, z, ql, z, 0.05, O.OracleConfig(**cfg))
    b = O.gp_flux(ql, z, ql, z, 0.05, O.OracleConfig(prandtl=0.72, **cfg))
    assert np.allclose(a["F"], b["F"], rtol=1e-13) and np.allclose(a["dF"], b["dF"], rtol=1e-12, atol=1e-14)
    a = O.gp_flux(ql, dql, qr, dqr, 0.05, O.OracleConfig())
    b = O.gp_flux(ql, dql, qr, dqr, 0.05, O.OracleConfig(prandtl=0.72))
    assert np.array_equal(a["F"], b["F"]) and np.array_equal(a["dF"], b["dF"])
