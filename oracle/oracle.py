"""ctypes front-end of the HGKS CPU oracle (oracle/hgks_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product
package (paper_2407_00656_b200) never imports it and shares no code with it.

Parity status per function:
  geometry, connectivity, stencils ........ pinned (closure, volumes, BFS, counts)
  least squares / WENO / beta ............. pinned (exactness, closed values, collapse)
  Maxwellian moments / micro-slopes ....... pinned (quadrature, numpy solve)
  Gauss-point GKS flux .................... pinned (brute-force quadrature of Eq. (flux),
                                             Euler limits, tau=0 Euler-chain identity)
  S2O4 stages ............................. pinned (Taylor polynomial of exp(z))
  full step ............................... pinned (conservation, free stream, T3 orders)
  farfield boundary state ................. pinned (characteristic conditions, seeded states)
  wall boundary state ..................... pinned (walled box: no mass/energy through the wall,
                                             closed-form no-slip stagnation pressure; test_oracle_wall.py)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hgks_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)


def build(force: bool = False) -> str:
    """Compile the oracle (plain -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
               "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.ora_last_error.restype = C.c_char_p
        L.ora_mesh_create.argtypes = [_dp, C.c_int64, _i8p, _i64p, C.c_int64, _dp, _dp, _i64p, _i32p, C.c_int64,
                                      C.POINTER(C.c_void_p)]
        L.ora_mesh_destroy.argtypes = [C.c_void_p]
        L.ora_mesh_counts.argtypes = [C.c_void_p, _i64p]
        L.ora_cell_geometry.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ora_faces.argtypes = [C.c_void_p, _i64p, _i64p, _i32p, _dp, _i32p, _dp, _dp, _dp]
        L.ora_cell_faces.argtypes = [C.c_void_p, _i64p]
        L.ora_big_stencil.argtypes = [C.c_void_p, C.c_int64, _i64p, _dp]
        L.ora_sub_stencil.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _i64p]
        L.ora_fit_cell.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, _dp, _dp, _dp, _dp]
        L.ora_weno_points.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, C.c_int64, _dp, _dp, _dp, C.c_int]
        L.ora_moments.argtypes = [_dp, C.c_double, C.c_int, _dp, _dp, _dp, _dp]
        L.ora_micro_slope.argtypes = [_dp, C.c_double, _dp, _dp]
        L.ora_slopes.argtypes = [_dp, C.c_double, _dp, _dp, _dp]
        L.ora_gp_flux.argtypes = [_dp, _dp, _dp, _dp, _dp, C.c_double, _dp]
        L.ora_local_frame.argtypes = [_dp, _dp, _dp]
        L.ora_farfield_state.argtypes = [_dp, _dp, _dp, _dp]
        L.ora_s2o4_stage1.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_double, _dp, _dp]
        L.ora_s2o4_stage2.argtypes = [C.c_int64, _dp, _dp, C.c_double, _dp]
        L.ora_solver_create.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.POINTER(C.c_void_p)]
        L.ora_solver_destroy.argtypes = [C.c_void_p]
        L.ora_solver_set_threads.argtypes = [C.c_void_p, C.c_int]
        L.ora_solver_step.argtypes = [C.c_void_p, C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.ora_solver_get.argtypes = [C.c_void_p, _dp, _dp, _dp, _i64p]
        L.ora_solver_set.argtypes = [C.c_void_p, _dp, C.c_double]
        L.ora_solver_dt.argtypes = [C.c_void_p]
        L.ora_solver_dt.restype = C.c_double
        L.ora_solver_residual.argtypes = [C.c_void_p, _dp, C.c_double, _dp, _dp, _i64p]
        _lib = L
    return _lib


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().ora_last_error().decode())


@dataclass
class OracleConfig:
    gamma: float = 1.4
    cfl: float = 0.3
    fixed_dt: float = 0.0
    tau_mode: int = 0          # 0: tau = 0 ; 1: Navier-Stokes tau (R7)
    c1: float = 1.0
    mu_inf: float = 0.0
    t_inf: float = 1.0
    mu_exp: float = 0.7
    eps: float = 1e-10
    omega_pow: int = 1
    freestream: tuple = (1.0, 0.0, 0.0, 0.0, 1.0 / 1.4)  # rho, U, V, W, p
    dq0_mode: int = 0          # equilibrium slopes: 0 average (R9), 1 kinetic (R9k), 2 gamma-weighted (R9s)
    prandtl: float = 1.0       # Pr != 1: heat-flux correction of the energy flux (R29)

    @property
    def K(self):
        return (5.0 - 3.0 * self.gamma) / (self.gamma - 1.0)

    def vec(self) -> np.ndarray:
        return np.array([self.gamma, self.cfl, self.fixed_dt, self.tau_mode, self.c1, self.mu_inf, self.t_inf,
                         self.mu_exp, self.eps, self.omega_pow, *self.freestream, self.dq0_mode, self.prandtl], dtype=np.float64)


class OracleMesh:
    def __init__(self, mi):
        L = lib()
        self.mi = mi
        xyz = np.ascontiguousarray(mi.xyz, np.float64)
        ct = np.ascontiguousarray(mi.cell_type, np.int8)
        cn = np.ascontiguousarray(mi.cell_nodes, np.int64)
        po = np.ascontiguousarray(mi.periodic_origin, np.float64)
        pl = np.ascontiguousarray(mi.periodic_length, np.float64)
        bf = np.ascontiguousarray(mi.bface_nodes, np.int64).reshape(-1, 4)
        bt = np.ascontiguousarray(mi.bface_tag, np.int32)
        h = C.c_void_p()
        _check(L.ora_mesh_create(_p(xyz), xyz.shape[0], _p(ct, _i8p), _p(cn, _i64p), cn.shape[0], _p(po), _p(pl),
                                 _p(bf, _i64p), _p(bt, _i32p), bf.shape[0], C.byref(h)))
        self.h = h
        c = np.zeros(6, np.int64)
        L.ora_mesh_counts(h, _p(c, _i64p))
        self.n_cells, self.n_faces, self.n_ghosts, self.max_stencil, self.min_stencil, self.n_subs = map(int, c)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_mesh_destroy(self.h)
            self.h = None

    def geometry(self):
        n = self.n_cells + self.n_ghosts
        V = np.zeros(n); c = np.zeros((n, 3)); M2 = np.zeros((n, 3, 3))
        lib().ora_cell_geometry(self.h, _p(V), _p(c), _p(M2))
        return V, c, M2

    def faces(self):
        nf = self.n_faces
        owner = np.zeros(nf, np.int64); nb = np.zeros(nf, np.int64); bc = np.zeros(nf, np.int32)
        shift = np.zeros((nf, 3)); ngp = np.zeros(nf, np.int32)
        gx = np.zeros((nf, 4, 3)); gn = np.zeros((nf, 4, 3)); gw = np.zeros((nf, 4))
        lib().ora_faces(self.h, _p(owner, _i64p), _p(nb, _i64p), _p(bc, _i32p), _p(shift), _p(ngp, _i32p),
                        _p(gx), _p(gn), _p(gw))
        return dict(owner=owner, nb=nb, bc=bc, shift=shift, ngp=ngp, gp_x=gx, gp_n=gn, gp_wS=gw)

    def cell_faces(self):
        cf = np.zeros((self.n_cells, 6), np.int64)
        lib().ora_cell_faces(self.h, _p(cf, _i64p))
        return cf

    def big_stencil(self, i):
        ids = np.zeros(128, np.int64); sh = np.zeros((128, 3))
        k = lib().ora_big_stencil(self.h, i, _p(ids, _i64p), _p(sh))
        return ids[:k].copy(), sh[:k].copy()

    def sub_stencil(self, i, m):
        ids = np.zeros(64, np.int64)
        k = lib().ora_sub_stencil(self.h, i, m, _p(ids, _i64p))
        return ids[:k].copy()

    def fit_cell(self, Q, i, cfg: OracleConfig | None = None):
        cfg = cfg or OracleConfig()
        Q = np.ascontiguousarray(Q, np.float64)
        a = np.zeros((9, 5)); b = np.zeros((8, 3, 5)); beta = np.zeros((9, 5)); wbar = np.zeros((9, 5))
        M = lib().ora_fit_cell(self.h, _p(cfg.vec()), _p(Q), i, _p(a), _p(b), _p(beta), _p(wbar))
        if M < 0:
            _check(-M)
        return dict(a=a, b=b[:M], beta=beta[:M + 1], wbar=wbar[:M + 1])

    def weno_points(self, Q, i, x, cfg: OracleConfig | None = None, linear: bool = False):
        """Eq. (weno) value and gradient of cell i at points x; linear=True uses the linear
        weights gamma in place of omega-bar (reading R9s)."""
        cfg = cfg or OracleConfig()
        Q = np.ascontiguousarray(Q, np.float64)
        x = np.ascontiguousarray(np.atleast_2d(x), np.float64)
        val = np.zeros((x.shape[0], 5)); grad = np.zeros((x.shape[0], 5, 3))
        _check(lib().ora_weno_points(self.h, _p(cfg.vec()), _p(Q), i, x.shape[0], _p(x), _p(val), _p(grad),
                                     1 if linear else 0))
        return val, grad


def moments(prim, K, rng):
    prim = np.ascontiguousarray(prim, np.float64)
    u = np.zeros(8); v = np.zeros(8); w = np.zeros(8); xi = np.zeros(3)
    lib().ora_moments(_p(prim), K, {"full": 0, "pos": 1, "neg": 2}[rng], _p(u), _p(v), _p(w), _p(xi))
    return u, v, w, xi


def micro_slope(q, K, b):
    q = np.ascontiguousarray(q, np.float64); b = np.ascontiguousarray(b, np.float64); a = np.zeros(5)
    lib().ora_micro_slope(_p(q), K, _p(b), _p(a))
    return a


def slopes(q, K, dq):
    q = np.ascontiguousarray(q, np.float64); dq = np.ascontiguousarray(dq, np.float64)
    a = np.zeros((3, 5)); A = np.zeros(5)
    lib().ora_slopes(_p(q), K, _p(dq), _p(a), _p(A))
    return a, A


def gp_flux(ql, dql, qr, dqr, dt, cfg: OracleConfig | None = None):
    """One Gauss point in the local frame.  Returns dict of I_half, I_full, F, dF, Q0, tau."""
    cfg = cfg or OracleConfig()
    arr = [np.ascontiguousarray(a, np.float64) for a in (ql, dql, qr, dqr)]
    out = np.zeros(41)
    lib().ora_gp_flux(_p(cfg.vec()), *[_p(a) for a in arr], dt, _p(out))
    return dict(I_half=out[0:5].copy(), I_full=out[5:10].copy(), F=out[10:15].copy(), dF=out[15:20].copy(),
                Q0=out[20:25].copy(), tau=float(out[25]), dq0=out[26:41].reshape(3, 5).copy())


def local_frame(n):
    n = np.ascontiguousarray(n, np.float64); t1 = np.zeros(3); t2 = np.zeros(3)
    lib().ora_local_frame(_p(n), _p(t1), _p(t2))
    return t1, t2


def farfield_state(qi, n, cfg: OracleConfig):
    qi = np.ascontiguousarray(qi, np.float64); n = np.ascontiguousarray(n, np.float64); qb = np.zeros(5)
    lib().ora_farfield_state(_p(cfg.vec()), _p(qi), _p(n), _p(qb))
    return qb


def s2o4_stage1(Qn, L, dL, dt):
    Qn, L, dL = [np.ascontiguousarray(a, np.float64) for a in (Qn, L, dL)]
    Qs = np.zeros_like(Qn); R = np.zeros_like(Qn)
    lib().ora_s2o4_stage1(Qn.size, _p(Qn), _p(L), _p(dL), dt, _p(Qs), _p(R))
    return Qs, R


def s2o4_stage2(R, dLs, dt):
    R, dLs = [np.ascontiguousarray(a, np.float64) for a in (R, dLs)]
    Q = np.zeros_like(R)
    lib().ora_s2o4_stage2(R.size, _p(R), _p(dLs), dt, _p(Q))
    return Q


class OracleSolver:
    def __init__(self, mesh: OracleMesh, Q0, cfg: OracleConfig | None = None, threads: int | None = None):
        self.mesh = mesh
        self.cfg = cfg or OracleConfig()
        Q0 = np.ascontiguousarray(Q0, np.float64)
        h = C.c_void_p()
        threads = threads or len(os.sched_getaffinity(0))
        self.threads = threads
        _check(lib().ora_solver_create(mesh.h, _p(self.cfg.vec()), _p(Q0), threads, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_solver_destroy(self.h)
            self.h = None

    def set_threads(self, n):
        self.threads = n
        lib().ora_solver_set_threads(self.h, n)

    def step(self, n_steps=1, t_stop=0.0):
        done = C.c_int(0)
        _check(lib().ora_solver_step(self.h, n_steps, t_stop, C.byref(done)))
        return done.value

    def state(self):
        Q = np.zeros((self.mesh.n_cells, 5)); t = C.c_double(); dt = C.c_double(); fb = C.c_int64()
        lib().ora_solver_get(self.h, _p(Q), C.byref(t), C.byref(dt), C.byref(fb))
        return Q, t.value, dt.value, fb.value

    def set_state(self, Q, t=0.0):
        Q = np.ascontiguousarray(Q, np.float64)
        lib().ora_solver_set(self.h, _p(Q), t)

    def dt(self):
        return lib().ora_solver_dt(self.h)

    def residual(self, Q, dt):
        Q = np.ascontiguousarray(Q, np.float64)
        L = np.zeros_like(Q); dL = np.zeros_like(Q); fb = C.c_int64()
        _check(lib().ora_solver_residual(self.h, _p(Q), dt, _p(L), _p(dL), C.byref(fb)))
        return L, dL, fb.value


def error_norms(rho_num, rho_exact, V, V_domain):
    """L1 = sum |e| V / V_D ; L2 = sqrt(sum e^2 V) / V_D (reading R22, pinned by T3's L1/L2 ratio)."""
    e = np.asarray(rho_num) - np.asarray(rho_exact)
    return float(np.sum(np.abs(e) * V) / V_domain), float(np.sqrt(np.sum(e * e * V)) / V_domain)
