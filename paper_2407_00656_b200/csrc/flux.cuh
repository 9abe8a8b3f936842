// a8 + a9: per Gauss point, evaluate both effective polynomials, rotate into
// the local frame, compute the BGK interface flux of Eq. (flux)
// and its time fit, rotate back and sum the face
// quadrature in Gauss-point order.  One thread per Gauss point;
// the per-face reduction goes through shared memory (deterministic, no atomics).
//
//   TAU0 = true : tau = 0, f = g0 (1 + A t) evaluated through the
//                 Euler-chain identity -- exact, ~1/3 the flops
//   TAU0 = false: full moment form with closed-form time integrals
//   BC = 0 interior, 1 no-slip wall (mirror), 2 farfield (Riemann) (R25)
#pragma once

// (included from kernels.cuh inside namespace hgks)

struct FluxArgs {
  const double* __restrict__ Q;  // [n_local][QS]
  const double* __restrict__ ceff;
  const int* __restrict__ f_cells;  // [n][2]
  const double* __restrict__ f_geo; // [n][stride]
  int f_stride;
  int n_faces;                      // faces in this launch
  int face0;                        // first face index
  double* __restrict__ F1;          // stage 1: [n_faces][10] (F*S, dF*S)
  double* __restrict__ F2;          // stage 2: [n_faces][5]  (dF*S)
  Ctrl* ctrl;
  GasParams gp;
};

// evaluate the effective polynomial of a cell at X (relative to its centroid)
// evaluate the effective polynomial of a cell at X (relative to its centroid);
// record layout rec[10 v + (const, x, y, z, xx, yy, zz, xy, xz, yz)], read as
// 16-byte vectors (80 bytes per variable)
__device__ __forceinline__ void eval_poly(const double* __restrict__ rec, const double X[3], double val[5],
                                          double grad[5][3]) {
  const double xx = X[0] * X[0], yy = X[1] * X[1], zz = X[2] * X[2];
  const double xy = X[0] * X[1], xz = X[0] * X[2], yz = X[1] * X[2];
  const double2* r2 = reinterpret_cast<const double2*>(rec);
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double2 a0 = __ldg(r2 + 5 * v), a1 = __ldg(r2 + 5 * v + 1), a2 = __ldg(r2 + 5 * v + 2),
                  a3 = __ldg(r2 + 5 * v + 3), a4 = __ldg(r2 + 5 * v + 4);
    const double c0 = a0.x, lx = a0.y, ly = a1.x, lz = a1.y, qxx = a2.x, qyy = a2.y, qzz = a3.x, qxy = a3.y,
                 qxz = a4.x, qyz = a4.y;
    val[v] = c0 + lx * X[0] + ly * X[1] + lz * X[2] + qxx * xx + qyy * yy + qzz * zz + qxy * xy + qxz * xz + qyz * yz;
    grad[v][0] = lx + 2.0 * qxx * X[0] + qxy * X[1] + qxz * X[2];
    grad[v][1] = ly + 2.0 * qyy * X[1] + qxy * X[0] + qyz * X[2];
    grad[v][2] = lz + 2.0 * qzz * X[2] + qxz * X[0] + qyz * X[1];
  }
}

// Gauss point g of a face from its vertices (relative to the owner centroid), R10
template <int NV>
__device__ __forceinline__ void face_gp(const double* __restrict__ fg, int g, double x[3], double n[3], double& wS) {
  if (NV == 3) {
    double p[3][3];
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int a = 0; a < 3; ++a) p[q][a] = __ldg(fg + 3 * q + a);
    const double e1[3] = {p[1][0] - p[0][0], p[1][1] - p[0][1], p[1][2] - p[0][2]};
    const double e2[3] = {p[2][0] - p[0][0], p[2][1] - p[0][1], p[2][2] - p[0][2]};
    double nn[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const double a2 = sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
    const double l0 = g == 0 ? 2.0 / 3.0 : 1.0 / 6.0, l1 = g == 1 ? 2.0 / 3.0 : 1.0 / 6.0,
                 l2 = g == 2 ? 2.0 / 3.0 : 1.0 / 6.0;
    const double ia = 1.0 / a2;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      x[a] = l0 * p[0][a] + l1 * p[1][a] + l2 * p[2][a];
      n[a] = nn[a] * ia;
    }
    wS = a2 * (1.0 / 6.0);
  } else {
    double p[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int a = 0; a < 3; ++a) p[q][a] = __ldg(fg + 3 * q + a);
    const double h = 0.28867513459481287;  // 1/(2 sqrt 3)
    const double s = (g & 1) ? 0.5 + h : 0.5 - h, t = (g >> 1) ? 0.5 + h : 0.5 - h;
    double ds[3], dt[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      x[a] = (1 - s) * (1 - t) * p[0][a] + s * (1 - t) * p[1][a] + s * t * p[2][a] + (1 - s) * t * p[3][a];
      ds[a] = (1 - t) * (p[1][a] - p[0][a]) + t * (p[2][a] - p[3][a]);
      dt[a] = (1 - s) * (p[3][a] - p[0][a]) + s * (p[2][a] - p[1][a]);
    }
    double nn[3] = {ds[1] * dt[2] - ds[2] * dt[1], ds[2] * dt[0] - ds[0] * dt[2], ds[0] * dt[1] - ds[1] * dt[0]};
    const double an = sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
    const double ia = 1.0 / an;
#pragma unroll
    for (int a = 0; a < 3; ++a) n[a] = nn[a] * ia;
    wS = 0.25 * an;
  }
}

// local frame (R11): t1 = normalize(n x e*), e* the axis with the smallest |n.e|
__device__ __forceinline__ void frame(const double n[3], double t1[3], double t2[3]) {
  int k = 0;
  if (fabs(n[1]) < fabs(n[k])) k = 1;
  if (fabs(n[2]) < fabs(n[k])) k = 2;
  double e[3] = {0.0, 0.0, 0.0};
  e[k] = 1.0;
  double c[3] = {n[1] * e[2] - n[2] * e[1], n[2] * e[0] - n[0] * e[2], n[0] * e[1] - n[1] * e[0]};
  double inv = 1.0 / sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
#pragma unroll
  for (int a = 0; a < 3; ++a) t1[a] = c[a] * inv;
  t2[0] = n[1] * t1[2] - n[2] * t1[1];
  t2[1] = n[2] * t1[0] - n[0] * t1[2];
  t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

// rotate value + gradient (global) into the local frame: q[5], dq[3][5] (derivative along n, t1, t2)
__device__ __forceinline__ void to_local(const double val[5], const double grad[5][3], const double n[3],
                                         const double t1[3], const double t2[3], double q[5], double dq[3][5]) {
  q[0] = val[0];
  q[4] = val[4];
  q[1] = val[1] * n[0] + val[2] * n[1] + val[3] * n[2];
  q[2] = val[1] * t1[0] + val[2] * t1[1] + val[3] * t1[2];
  q[3] = val[1] * t2[0] + val[2] * t2[1] + val[3] * t2[2];
  // frame matrix rows (n, t1, t2), indexed with compile-time j only (stays in registers)
  const double Rm[3][3] = {{n[0], n[1], n[2]}, {t1[0], t1[1], t1[2]}, {t2[0], t2[1], t2[2]}};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double* e = Rm[j];
    double d[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) d[v] = grad[v][0] * e[0] + grad[v][1] * e[1] + grad[v][2] * e[2];
    dq[j][0] = d[0];
    dq[j][4] = d[4];
    dq[j][1] = d[1] * n[0] + d[2] * n[1] + d[3] * n[2];
    dq[j][2] = d[1] * t1[0] + d[2] * t1[1] + d[3] * t1[2];
    dq[j][3] = d[1] * t2[0] + d[2] * t2[1] + d[3] * t2[2];
  }
}

// Euler-flux Jacobian-vector product along local axis j: dF_j = (dF_j/dQ) dq
// Euler state quantities shared by the Jacobian-vector products below
struct EulerState {
  double Q[5], inv, u[3], p, H, q2h;  // H = rhoE + p, q2h = |u|^2 / 2
};
__device__ __forceinline__ EulerState euler_state(const double Q[5], double gm1) {
  EulerState e;
#pragma unroll
  for (int v = 0; v < 5; ++v) e.Q[v] = Q[v];
  e.inv = 1.0 / Q[0];
  e.u[0] = Q[1] * e.inv;
  e.u[1] = Q[2] * e.inv;
  e.u[2] = Q[3] * e.inv;
  e.q2h = 0.5 * (e.u[0] * e.u[0] + e.u[1] * e.u[1] + e.u[2] * e.u[2]);
  e.p = gm1 * (Q[4] - Q[0] * e.q2h);
  e.H = Q[4] + e.p;
  return e;
}
// Euler-flux Jacobian-vector product along local axis j: dF_j = (dF_j/dQ) dq
__device__ __forceinline__ void euler_jvp(int j, const EulerState& e, const double dq[5], double gm1, double out[5]) {
  const double du[3] = {(dq[1] - e.u[0] * dq[0]) * e.inv, (dq[2] - e.u[1] * dq[0]) * e.inv,
                        (dq[3] - e.u[2] * dq[0]) * e.inv};
  const double dp = gm1 * (dq[4] - (e.u[0] * dq[1] + e.u[1] * dq[2] + e.u[2] * dq[3]) + e.q2h * dq[0]);
  out[0] = dq[1 + j];
#pragma unroll
  for (int k = 0; k < 3; ++k) out[1 + k] = dq[1 + j] * e.u[k] + e.Q[1 + j] * du[k] + (k == j ? dp : 0.0);
  out[4] = du[j] * e.H + e.u[j] * (dq[4] + dp);
}


// ---------------------------------------------------------------------------
// Moment form (general tau).  Moments of a Maxwellian normalised by rho:
// <u^a> (full line, u>0 or u<0), <v^b>, <w^c> (full), <xi^2>, <xi^4>
// (SURVEY A.1).  psi = (1, u, v, w, (u^2+v^2+w^2+xi^2)/2).
// ---------------------------------------------------------------------------
struct Mom {
  double U[7], V[6], W[6], X1, X2;
};

// full moments of v, w and xi; u moments over RANGE (0 full, 1 u>0, 2 u<0)
template <int RANGE>
__device__ __forceinline__ void maxwell_moments(double U, double V, double W, double lam, double K, Mom& m) {
  const double h = 0.5 / lam;  // 1/(2 lambda)
  if (RANGE == 0) {
    m.U[0] = 1.0;
    m.U[1] = U;
  } else {
    const double sl = sqrt(lam);
    const double e = 0.5 * exp(-lam * U * U) * 0.56418958354775628 / sl;  // e^{-lam U^2} / (2 sqrt(pi lam))
    if (RANGE == 1) {
      m.U[0] = 0.5 * erfc(-sl * U);
      m.U[1] = U * m.U[0] + e;
    } else {
      m.U[0] = 0.5 * erfc(sl * U);
      m.U[1] = U * m.U[0] - e;
    }
  }
#pragma unroll
  for (int n = 0; n < 5; ++n) m.U[n + 2] = U * m.U[n + 1] + (n + 1) * h * m.U[n];
  m.V[0] = 1.0;
  m.V[1] = V;
  m.W[0] = 1.0;
  m.W[1] = W;
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    m.V[n + 2] = V * m.V[n + 1] + (n + 1) * h * m.V[n];
    m.W[n + 2] = W * m.W[n + 1] + (n + 1) * h * m.W[n];
  }
  m.X1 = K * h;
  m.X2 = K * (K + 2.0) * h * h;
}

// <u^A v^B w^C psi>
template <int A, int B, int C>
__device__ __forceinline__ void psi_m(const Mom& m, double o[5]) {
  const double uvw = m.U[A] * m.V[B] * m.W[C];
  o[0] = uvw;
  o[1] = m.U[A + 1] * m.V[B] * m.W[C];
  o[2] = m.U[A] * m.V[B + 1] * m.W[C];
  o[3] = m.U[A] * m.V[B] * m.W[C + 1];
  o[4] = 0.5 * (m.U[A + 2] * m.V[B] * m.W[C] + m.U[A] * m.V[B + 2] * m.W[C] + m.U[A] * m.V[B] * m.W[C + 2] + uvw * m.X1);
}
// <u^A v^B w^C xi^2 psi>
template <int A, int B, int C>
__device__ __forceinline__ void psi_mx(const Mom& m, double o[5]) {
  const double uvw = m.U[A] * m.V[B] * m.W[C];
  o[0] = uvw * m.X1;
  o[1] = m.U[A + 1] * m.V[B] * m.W[C] * m.X1;
  o[2] = m.U[A] * m.V[B + 1] * m.W[C] * m.X1;
  o[3] = m.U[A] * m.V[B] * m.W[C + 1] * m.X1;
  o[4] = 0.5 * (m.X1 * (m.U[A + 2] * m.V[B] * m.W[C] + m.U[A] * m.V[B + 2] * m.W[C] + m.U[A] * m.V[B] * m.W[C + 2]) +
                uvw * m.X2);
}
// <s u^A v^B w^C psi> for a slope s = s0 + s1 u + s2 v + s3 w + s4 psi_5
template <int A, int B, int C>
__device__ __forceinline__ void slope_m(const Mom& m, const double s[5], double o[5]) {
  double t[5];
  psi_m<A, B, C>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = s[0] * t[k];
  psi_m<A + 1, B, C>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(s[1], t[k], o[k]);
  psi_m<A, B + 1, C>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(s[2], t[k], o[k]);
  psi_m<A, B, C + 1>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(s[3], t[k], o[k]);
  const double h4 = 0.5 * s[4];
  psi_m<A + 2, B, C>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(h4, t[k], o[k]);
  psi_m<A, B + 2, C>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(h4, t[k], o[k]);
  psi_m<A, B, C + 2>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(h4, t[k], o[k]);
  psi_mx<A, B, C>(m, t);
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = fma(h4, t[k], o[k]);
}

// micro-slope a with sum_j a_j <psi_i psi_j> = b_i (b already divided by rho),
// closed form of the 5x5 Maxwellian moment system
__device__ __forceinline__ void micro_slope(const double b[5], double U, double V, double W, double lam, double K,
                                            double a[5]) {
  const double B = U * U + V * V + W * W + (K + 3.0) / (2.0 * lam);
  const double R1 = b[1] - U * b[0], R2 = b[2] - V * b[0], R3 = b[3] - W * b[0];
  const double R4 = 2.0 * b[4] - B * b[0];
  a[4] = 4.0 * lam * lam / (K + 3.0) * (R4 - 2.0 * U * R1 - 2.0 * V * R2 - 2.0 * W * R3);
  a[1] = 2.0 * lam * R1 - U * a[4];
  a[2] = 2.0 * lam * R2 - V * a[4];
  a[3] = 2.0 * lam * R3 - W * a[4];
  a[0] = b[0] - U * a[1] - V * a[2] - W * a[3] - 0.5 * a[4] * B;
}

struct Prim {
  double rho, U, V, W, lam;
};
__device__ __forceinline__ Prim prim_of(const double q[5], double K) {
  Prim p;
  p.rho = q[0];
  const double inv = 1.0 / q[0];
  p.U = q[1] * inv;
  p.V = q[2] * inv;
  p.W = q[3] * inv;
  p.lam = (K + 3.0) * p.rho / (4.0 * (q[4] - 0.5 * p.rho * (p.U * p.U + p.V * p.V + p.W * p.W)));
  return p;
}


// closed-form time integrals of the Eq. (flux) coefficients over [0, delta]
struct TimeCoef {
  double c1, c2, c3, c4, c5, c6;
};
__device__ __forceinline__ TimeCoef time_coef(double delta, double tau) {
  TimeCoef c;
  const double e = exp(-delta / tau);
  const double om = 1.0 - e;
  c.c1 = delta - tau * om;
  c.c2 = 2.0 * tau * tau * om - tau * delta * (1.0 + e);
  c.c3 = 0.5 * delta * delta - tau * delta + tau * tau * om;
  c.c4 = tau * om;
  c.c5 = -2.0 * tau * tau * om + tau * delta * e;
  c.c6 = -tau * tau * om;
  return c;
}

// Q0 = int_{u>0} psi g_l + int_{u<0} psi g_r
__device__ __forceinline__ void equilibrium_state(const double ql[5], const double qr[5], double K, double Q0[5]) {
  const double rpi = 0.56418958354775628;  // 1/sqrt(pi)
  const Prim l = prim_of(ql, K), r = prim_of(qr, K);
  const double hl = 0.5 / l.lam, hr = 0.5 / r.lam;  // 1/(2 lambda)
  const double isl = rsqrt(l.lam), isr = rsqrt(r.lam);
  const double a0 = 0.5 * erfc(-(l.lam * isl) * l.U);
  const double a1 = l.U * a0 + 0.5 * exp(-l.lam * l.U * l.U) * rpi * isl;
  const double a2 = l.U * a1 + a0 * hl;
  const double b0 = 0.5 * erfc((r.lam * isr) * r.U);
  const double b1 = r.U * b0 - 0.5 * exp(-r.lam * r.U * r.U) * rpi * isr;
  const double b2 = r.U * b1 + b0 * hr;
  Q0[0] = l.rho * a0 + r.rho * b0;
  Q0[1] = l.rho * a1 + r.rho * b1;
  Q0[2] = l.rho * a0 * l.V + r.rho * b0 * r.V;
  Q0[3] = l.rho * a0 * l.W + r.rho * b0 * r.W;
  Q0[4] = 0.5 * l.rho * (a2 + a0 * (l.V * l.V + l.W * l.W + (K + 2.0) * hl)) +
          0.5 * r.rho * (b2 + b0 * (r.V * r.V + r.W * r.W + (K + 2.0) * hr));
}

// One term group of Eq. (flux) for a Maxwellian with its slopes, accumulated into
// I_half, I_full (rho-weighted).  Full-range Maxwellian moments of the slope
// polynomials reduce to Euler-flux Jacobian-vector products (d_j g = a_j g, so
// rho <u_j a_j psi> = A_j(Q) d_j Q): the compatibility condition
// for A becomes d_t Q = -sum_j A_j(Q) d_j Q, and for the equilibrium
// part rho<u psi> = F_n(Q), rho<A u psi> = A_n(Q) d_t Q.  Only <(a.u) u psi>
// (full range for g0) and the half-range moments of g_l, g_r need the generic
// moment sums.
template <int RANGE>
__device__ __forceinline__ void add_side(const double q[5], const double dq[3][5], double K, double gm1,
                                         const TimeCoef& ch, const TimeCoef& cf, double Ih[5], double If[5]) {
  const Prim g = prim_of(q, K);
  const double ir = 1.0 / g.rho;
  double a[3][5];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    double b[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) b[v] = dq[j][v] * ir;
    micro_slope(b, g.U, g.V, g.W, g.lam, K, a[j]);
  }
  const EulerState es = euler_state(q, gm1);
  double dtq[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // d_t Q by compatibility
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    double jv[5];
    euler_jvp(j, es, dq[j], gm1, jv);
#pragma unroll
    for (int v = 0; v < 5; ++v) dtq[v] -= jv[v];
  }
  Mom mom;
  maxwell_moments<RANGE>(g.U, g.V, g.W, g.lam, K, mom);
  double m2[5];  // <(a.u) u psi> over the range
  {
    double t0[5], t1[5], t2[5];
    slope_m<2, 0, 0>(mom, a[0], t0);
    slope_m<1, 1, 0>(mom, a[1], t1);
    slope_m<1, 0, 1>(mom, a[2], t2);
#pragma unroll
    for (int v = 0; v < 5; ++v) m2[v] = g.rho * (t0[v] + t1[v] + t2[v]);
  }
  if (RANGE == 0) {
    // rho <u psi> = F_n(Q) and rho <A u psi> = A_n(Q) d_t Q
    double m3[5];
    euler_jvp(0, es, dtq, gm1, m3);
    const double m1[5] = {q[1], q[1] * es.u[0] + es.p, q[2] * es.u[0], q[3] * es.u[0], es.u[0] * es.H};
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      Ih[v] += ch.c1 * m1[v] + ch.c2 * m2[v] + ch.c3 * m3[v];
      If[v] += cf.c1 * m1[v] + cf.c2 * m2[v] + cf.c3 * m3[v];
    }
  } else {
    double A[5], b[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) b[v] = dtq[v] * ir;
    micro_slope(b, g.U, g.V, g.W, g.lam, K, A);
    double m1[5], m3[5];
    psi_m<1, 0, 0>(mom, m1);
    slope_m<1, 0, 0>(mom, A, m3);
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      Ih[v] += g.rho * (ch.c4 * m1[v] + ch.c6 * m3[v]) + ch.c5 * m2[v];
      If[v] += g.rho * (cf.c4 * m1[v] + cf.c6 * m3[v]) + cf.c5 * m2[v];
    }
  }
}

// boundary right states in the local frame (R25)
template <int BC>
__device__ __forceinline__ void boundary_right(const double ql[5], const double dql[3][5], const double vl_global[5],
                                               const double n[3], const double t1[3], const double t2[3],
                                               const GasParams& gp, double qr[5], double dqr[3][5]) {
  if (BC == 1) {  // wall mirror: all velocity components reversed, normal derivatives negated
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double sv = (v >= 1 && v <= 3) ? -1.0 : 1.0;
      qr[v] = sv * ql[v];
      dqr[0][v] = -sv * dql[0][v];
      dqr[1][v] = sv * dql[1][v];
      dqr[2][v] = sv * dql[2][v];
    }
  } else {  // farfield: Riemann state of the left value, zero gradient
    double qb[5];
    farfield_riemann(vl_global, n, gp, qb);
    qr[0] = qb[0];
    qr[4] = qb[4];
    qr[1] = qb[1] * n[0] + qb[2] * n[1] + qb[3] * n[2];
    qr[2] = qb[1] * t1[0] + qb[2] * t1[1] + qb[3] * t1[2];
    qr[3] = qb[1] * t2[0] + qb[2] * t2[1] + qb[3] * t2[2];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int v = 0; v < 5; ++v) dqr[j][v] = 0.0;
  }
}

template <int NV, int STAGE, bool TAU0, int BC>
__global__ void __launch_bounds__(NV == 3 ? 96 : 128, TAU0 ? (NV == 3 ? 5 : 4) : 1) k_flux(FluxArgs a) {
  constexpr int NGP = NV == 3 ? 3 : 4;
  constexpr int BLOCK = NV == 3 ? 96 : 128;
  constexpr int NOUT = STAGE == 1 ? 10 : 5;
  __shared__ double red[NOUT][BLOCK];
  const int t = blockIdx.x * BLOCK + threadIdx.x;
  const int lf = t / NGP, g = t - lf * NGP;
  const bool active = lf < a.n_faces;
  double out[NOUT];
#pragma unroll
  for (int k = 0; k < NOUT; ++k) out[k] = 0.0;
  if (active) {
    const int f = a.face0 + lf;
    const int co = __ldg(a.f_cells + 2 * f);
    const double* fg = a.f_geo + (size_t)f * a.f_stride;
    double x[3], n[3], wS;
    face_gp<NV>(fg, g, x, n, wS);
    double t1[3], t2[3];
    frame(n, t1, t2);
    const double K = a.gp.K;
    const double gm1 = a.gp.gamma - 1.0;
    // positivity check without a division: for rho > 0, p > 0  <=>  rho*rhoE - |m|^2/2 > 0 (R21)
    auto admissible = [](const double q[5]) {
      return q[0] > 0.0 && (q[0] * q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3])) > 0.0;
    };
    auto rotate_value = [&](const double v5[5], double q[5]) {
      q[0] = v5[0];
      q[4] = v5[4];
      q[1] = v5[1] * n[0] + v5[2] * n[1] + v5[3] * n[2];
      q[2] = v5[1] * t1[0] + v5[2] * t1[1] + v5[3] * t1[2];
      q[3] = v5[1] * t2[0] + v5[2] * t2[1] + v5[3] * t2[2];
    };
    double F[5], dF[5];
    if (TAU0 && BC == 0) {
      // tau = 0 interior face: only the average of the two gradients enters (R9),
      // so it is summed in the global frame and rotated once
      double ql[5], qr[5], gs[5][3];
      {
        double vl[5];
        eval_poly(a.ceff + (size_t)co * kRec, x, vl, gs);
        if (!admissible(vl)) {
          atomicAdd((unsigned long long*)&a.ctrl->fallbacks, 1ull);
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            vl[v] = a.Q[(size_t)co * QS + v];
            gs[v][0] = gs[v][1] = gs[v][2] = 0.0;
          }
        }
        rotate_value(vl, ql);
      }
      {
        const int cn = __ldg(a.f_cells + 2 * f + 1);
        const double xr[3] = {x[0] + __ldg(fg + 3 * NV), x[1] + __ldg(fg + 3 * NV + 1),
                              x[2] + __ldg(fg + 3 * NV + 2)};
        double vr[5], gr[5][3];
        eval_poly(a.ceff + (size_t)cn * kRec, xr, vr, gr);
        if (!admissible(vr)) {
          atomicAdd((unsigned long long*)&a.ctrl->fallbacks, 1ull);
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            vr[v] = a.Q[(size_t)cn * QS + v];
            gr[v][0] = gr[v][1] = gr[v][2] = 0.0;
          }
        }
        rotate_value(vr, qr);
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int c = 0; c < 3; ++c) gs[v][c] = 0.5 * (gs[v][c] + gr[v][c]);
      }
      double dq0[3][5];
      {
        double zero[5] = {0, 0, 0, 0, 0}, dummy[5];
        to_local(zero, gs, n, t1, t2, dummy, dq0);
      }
      double Q0[5];
      equilibrium_state(ql, qr, K, Q0);
      // f = g0 (1 + A t): F = Euler flux of Q0, d_t F = A_n(Q0) d_t Q0,
      // d_t Q0 = -sum_j A_j(Q0) d_j Q0
      const EulerState es = euler_state(Q0, gm1);
      double dtQ0[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double jv[5];
        euler_jvp(j, es, dq0[j], gm1, jv);
#pragma unroll
        for (int v = 0; v < 5; ++v) dtQ0[v] -= jv[v];
      }
      euler_jvp(0, es, dtQ0, gm1, dF);
      F[0] = Q0[1];
      F[1] = Q0[1] * es.u[0] + es.p;
      F[2] = Q0[2] * es.u[0];
      F[3] = Q0[3] * es.u[0];
      F[4] = es.u[0] * es.H;
    } else {
    double ql[5], dql[3][5], qr[5], dqr[3][5];
    double vl[5];
    {
      double grad[5][3];
      eval_poly(a.ceff + (size_t)co * kRec, x, vl, grad);
      if (!admissible(vl)) {  // R21 positivity fallback
        atomicAdd((unsigned long long*)&a.ctrl->fallbacks, 1ull);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          vl[v] = a.Q[(size_t)co * QS + v];
          grad[v][0] = grad[v][1] = grad[v][2] = 0.0;
        }
      }
      to_local(vl, grad, n, t1, t2, ql, dql);
    }
    if (BC == 0) {
      const int cn = __ldg(a.f_cells + 2 * f + 1);
      const double xr[3] = {x[0] + __ldg(fg + 3 * NV), x[1] + __ldg(fg + 3 * NV + 1), x[2] + __ldg(fg + 3 * NV + 2)};
      double val[5], grad[5][3];
      eval_poly(a.ceff + (size_t)cn * kRec, xr, val, grad);
      if (!admissible(val)) {
        atomicAdd((unsigned long long*)&a.ctrl->fallbacks, 1ull);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          val[v] = a.Q[(size_t)cn * QS + v];
          grad[v][0] = grad[v][1] = grad[v][2] = 0.0;
        }
      }
      to_local(val, grad, n, t1, t2, qr, dqr);
    } else {
      boundary_right<BC>(ql, dql, vl, n, t1, t2, a.gp, qr, dqr);
    }
    double Q0[5];
    equilibrium_state(ql, qr, K, Q0);
    if (TAU0) {
      double dtQ0[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      const EulerState es = euler_state(Q0, gm1);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double d0[5], jv[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) d0[v] = 0.5 * (dql[j][v] + dqr[j][v]);
        euler_jvp(j, es, d0, gm1, jv);
#pragma unroll
        for (int v = 0; v < 5; ++v) dtQ0[v] -= jv[v];
      }
      euler_jvp(0, es, dtQ0, gm1, dF);
      F[0] = Q0[1];
      F[1] = Q0[1] * es.u[0] + es.p;
      F[2] = Q0[2] * es.u[0];
      F[3] = Q0[3] * es.u[0];
      F[4] = es.u[0] * es.H;
    } else {
      // collision time (R7): tau = mu(T0)/p0 + c1 |pl - pr|/(pl + pr) dt
      const double dt = a.ctrl->dt;
      const Prim g0 = prim_of(Q0, K), gl = prim_of(ql, K), gr = prim_of(qr, K);
      const double p0 = g0.rho / (2.0 * g0.lam), pl = gl.rho / (2.0 * gl.lam), pr = gr.rho / (2.0 * gr.lam);
      const double mu = a.gp.mu_inf * pow((p0 / g0.rho) / a.gp.t_inf, a.gp.mu_exp);
      const double tau = mu / p0 + a.gp.c1 * fabs(pl - pr) / (pl + pr) * dt;
      const TimeCoef ch = time_coef(0.5 * dt, tau), cf = time_coef(dt, tau);
      double Ih[5] = {0, 0, 0, 0, 0}, If[5] = {0, 0, 0, 0, 0};
      double dq0[3][5];
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int v = 0; v < 5; ++v) dq0[j][v] = 0.5 * (dql[j][v] + dqr[j][v]);
      add_side<0>(Q0, dq0, K, gm1, ch, cf, Ih, If);
      add_side<1>(ql, dql, K, gm1, ch, cf, Ih, If);
      add_side<2>(qr, dqr, K, gm1, ch, cf, Ih, If);
      // 2x2 fit
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        F[v] = (4.0 * Ih[v] - If[v]) / dt;
        dF[v] = 4.0 * (If[v] - 2.0 * Ih[v]) / (dt * dt);
      }
    }
    }
    // rotate back to the global frame and weight by omega_G S
    if (STAGE == 1) {
      out[0] = wS * F[0];
#pragma unroll
      for (int c = 0; c < 3; ++c) out[1 + c] = wS * (F[1] * n[c] + F[2] * t1[c] + F[3] * t2[c]);
      out[4] = wS * F[4];
      out[5] = wS * dF[0];
#pragma unroll
      for (int c = 0; c < 3; ++c) out[6 + c] = wS * (dF[1] * n[c] + dF[2] * t1[c] + dF[3] * t2[c]);
      out[9] = wS * dF[4];
    } else {
      out[0] = wS * dF[0];
#pragma unroll
      for (int c = 0; c < 3; ++c) out[1 + c] = wS * (dF[1] * n[c] + dF[2] * t1[c] + dF[3] * t2[c]);
      out[4] = wS * dF[4];
    }
  }
#pragma unroll
  for (int k = 0; k < NOUT; ++k) red[k][threadIdx.x] = out[k];
  __syncthreads();
  // face quadrature sum in Gauss-point order (deterministic)
  const int faces_in_block = BLOCK / NGP;
  for (int e = threadIdx.x; e < faces_in_block * NOUT; e += BLOCK) {
    const int fl = e / NOUT, k = e - fl * NOUT;
    const int face = blockIdx.x * faces_in_block + fl;
    if (face < a.n_faces) {
      double s = red[k][fl * NGP];
#pragma unroll
      for (int q = 1; q < NGP; ++q) s += red[k][fl * NGP + q];
      double* dst = STAGE == 1 ? a.F1 : a.F2;
      dst[(size_t)(a.face0 + face) * NOUT + k] = s;
    }
  }
}


