// Algorithmic flop count of one interior-face flux of the tau = 0 path and
// of the tau > 0 moment form per Gauss point is NOT done here; this counts the tau = 0
// reduced form only, for the roofline of k_flux tau0 (bench.py "flops_source").
//
// A plain evaluation of the formulas with an operation-counting scalar: + - * / each one
// flop, fma two, sqrt / exp / erfc one each (a transcendental counts as one operation, the
// convention of an algorithmic count; the kernel's own polynomial erfc/exp cost more).
// Per interior triangle face: the face normal and local frame once (planar triangle), then
// per Gauss point (3): both cells' effective quadratics (value + gradient) at the point,
// rotation into (n, t1, t2), the equilibrium state Q0 from the two half-range Maxwellian
// moment sets, F = Euler flux of Q0, d_t F = A_n(Q0)(-sum_j A_j(Q0) d_j Q0) with
// d_j Q0 = average of the two gradients (R9), rotation back, weight; the 3-point face sum.
//
//   g++ -O1 -std=c++17 tools/flop_count/flux_tau0_flops.cpp -o /tmp/ffc && /tmp/ffc
// (result recorded in profiles/flops_algorithmic.json)
#include <cmath>
#include <cstdio>

static long long g_flops = 0;
struct F {
  double v;
  F(double x = 0) : v(x) {}
};
F operator+(F a, F b) { ++g_flops; return a.v + b.v; }
F operator-(F a, F b) { ++g_flops; return a.v - b.v; }
F operator*(F a, F b) { ++g_flops; return a.v * b.v; }
F operator/(F a, F b) { ++g_flops; return a.v / b.v; }
F operator-(F a) { return -a.v; }  // sign flip: free
F& operator+=(F& a, F b) { a = a + b; return a; }
F& operator-=(F& a, F b) { a = a - b; return a; }
F fsqrt(F a) { ++g_flops; return std::sqrt(a.v); }
F fexp(F a) { ++g_flops; return std::exp(a.v); }
F ferfc(F a) { ++g_flops; return std::erfc(a.v); }

const double K = 2.0, gam = 1.4;

// quadratic record (const, lin[3], quad xx yy zz xy xz yz) per variable at X
void eval(const F c[5][10], const F X[3], F val[5], F grad[5][3]) {
  F xx = X[0] * X[0], yy = X[1] * X[1], zz = X[2] * X[2], xy = X[0] * X[1], xz = X[0] * X[2], yz = X[1] * X[2];
  for (int v = 0; v < 5; ++v) {
    val[v] = c[v][0] + c[v][1] * X[0] + c[v][2] * X[1] + c[v][3] * X[2] + c[v][4] * xx + c[v][5] * yy +
             c[v][6] * zz + c[v][7] * xy + c[v][8] * xz + c[v][9] * yz;
    grad[v][0] = c[v][1] + F(2.0) * c[v][4] * X[0] + c[v][7] * X[1] + c[v][8] * X[2];
    grad[v][1] = c[v][2] + F(2.0) * c[v][5] * X[1] + c[v][7] * X[0] + c[v][9] * X[2];
    grad[v][2] = c[v][3] + F(2.0) * c[v][6] * X[2] + c[v][8] * X[0] + c[v][9] * X[1];
  }
}
F dot3(const F a[3], const F b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
void rot(const F m[3], const F R[3][3], F o[3]) { for (int j = 0; j < 3; ++j) o[j] = dot3(m, R[j]); }

// rho <psi>_{u>0 or u<0} of a Maxwellian given by conserved q (local frame)
void half(const F q[5], double sg, F out[5]) {
  F rho = q[0], U = q[1] / rho, V = q[2] / rho, W = q[3] / rho;
  F p = F(gam - 1) * (q[4] - F(0.5) * rho * (U * U + V * V + W * W));
  F lam = rho / (F(2.0) * p);
  F sl = fsqrt(lam);
  F m0 = F(0.5) * ferfc(F(-sg) * sl * U);
  F e = fexp(-(lam * U * U)) / (F(2.0) * fsqrt(F(M_PI) * lam));
  F m1 = U * m0 + F(sg) * e;
  F m2 = U * m1 + m0 / (F(2.0) * lam);
  out[0] = rho * m0;
  out[1] = rho * m1;
  out[2] = rho * m0 * V;
  out[3] = rho * m0 * W;
  out[4] = F(0.5) * rho * (m2 + m0 * (V * V + W * W + F(K) / (F(2.0) * lam)));
}
// Euler state of Q0 (computed once per Gauss point) and the Jacobian-vector product of the
// Euler flux along local axis j
struct ES {
  F ir, u[3], q2, p, H;
};
ES estate(const F Q[5]) {
  ES e;
  e.ir = F(1.0) / Q[0];
  for (int k = 0; k < 3; ++k) e.u[k] = Q[1 + k] * e.ir;
  e.q2 = F(0.5) * (e.u[0] * e.u[0] + e.u[1] * e.u[1] + e.u[2] * e.u[2]);
  e.p = F(gam - 1) * (Q[4] - Q[0] * e.q2);
  e.H = Q[4] + e.p;
  return e;
}
void jvp(int j, const F Q[5], const ES& e, const F dq[5], F out[5]) {
  const F ir = e.ir, q2 = e.q2, H = e.H;
  const F* u = e.u;
  F du[3];
  for (int k = 0; k < 3; ++k) du[k] = (dq[1 + k] - u[k] * dq[0]) * ir;
  F dp = F(gam - 1) * (dq[4] - (u[0] * dq[1] + u[1] * dq[2] + u[2] * dq[3]) + q2 * dq[0]);
  out[0] = dq[1 + j];
  for (int k = 0; k < 3; ++k) out[1 + k] = dq[1 + j] * u[k] + Q[1 + j] * du[k] + (k == j ? dp : F(0.0));
  out[4] = du[j] * H + u[j] * (dq[4] + dp);
}

long long face_flops(int stage);
int main() {
  const long long s1 = face_flops(1), s2 = face_flops(2);
  std::printf("{\"per_face_stage1\": %lld, \"per_face_stage2\": %lld}\n", s1, s2);
  return 0;
}

long long face_flops(int stage) {
  F cl[5][10], cr[5][10], vtx[3][3], d[3];
  for (int v = 0; v < 5; ++v)
    for (int k = 0; k < 10; ++k) { cl[v][k] = 0.01 * (k + 1); cr[v][k] = 0.02 * (k + 1); }
  cl[0][0] = cr[0][0] = 1.0; cl[4][0] = cr[4][0] = 3.0;
  double P[3][3] = {{0.1, 0.0, 0.0}, {0.0, 0.1, 0.0}, {0.0, 0.0, 0.1}};
  for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) vtx[a][b] = P[a][b];
  d[0] = 0.05; d[1] = 0.05; d[2] = 0.05;
  g_flops = 0;
  // per face: normal (cross product), area, frame
  F e1[3], e2[3], nn[3];
  for (int a = 0; a < 3; ++a) { e1[a] = vtx[1][a] - vtx[0][a]; e2[a] = vtx[2][a] - vtx[0][a]; }
  nn[0] = e1[1] * e2[2] - e1[2] * e2[1]; nn[1] = e1[2] * e2[0] - e1[0] * e2[2]; nn[2] = e1[0] * e2[1] - e1[1] * e2[0];
  F a2 = fsqrt(dot3(nn, nn)), ia = F(1.0) / a2, wS = a2 / F(6.0);
  F n[3] = {nn[0] * ia, nn[1] * ia, nn[2] * ia};
  F c[3] = {n[1], -n[0], F(0.0)};  // n x e_z (the axis choice is a comparison, no flops)
  F ic = F(1.0) / fsqrt(c[0] * c[0] + c[1] * c[1]);
  F t1[3] = {c[0] * ic, c[1] * ic, F(0.0)};
  F t2[3] = {n[1] * t1[2] - n[2] * t1[1], n[2] * t1[0] - n[0] * t1[2], n[0] * t1[1] - n[1] * t1[0]};
  F R[3][3] = {{n[0], n[1], n[2]}, {t1[0], t1[1], t1[2]}, {t2[0], t2[1], t2[2]}};
  long long face_part = g_flops;
  F sum[10];
  for (int g = 0; g < 3; ++g) {
    F X[3], Xr[3];
    for (int a = 0; a < 3; ++a) {
      X[a] = F(2.0 / 3.0) * vtx[g][a] + F(1.0 / 6.0) * (vtx[(g + 1) % 3][a] + vtx[(g + 2) % 3][a]);
      Xr[a] = X[a] + d[a];
    }
    F vl[5], gl[5][3], vr[5], gr[5][3];
    eval(cl, X, vl, gl);
    eval(cr, Xr, vr, gr);
    F ql[5], qr[5], m[3];
    ql[0] = vl[0]; ql[4] = vl[4]; qr[0] = vr[0]; qr[4] = vr[4];
    { F mm[3] = {vl[1], vl[2], vl[3]}; rot(mm, R, m); for (int k = 0; k < 3; ++k) ql[1 + k] = m[k]; }
    { F mm[3] = {vr[1], vr[2], vr[3]}; rot(mm, R, m); for (int k = 0; k < 3; ++k) qr[1 + k] = m[k]; }
    // dQ0 = (grad_l + grad_r)/2 along n, t1, t2, momentum rotated
    F dq0[3][5];
    for (int j = 0; j < 3; ++j) {
      F dd[5];
      for (int v = 0; v < 5; ++v) dd[v] = F(0.5) * (dot3(gl[v], R[j]) + dot3(gr[v], R[j]));
      F mm[3] = {dd[1], dd[2], dd[3]};
      rot(mm, R, m);
      dq0[j][0] = dd[0]; dq0[j][4] = dd[4];
      for (int k = 0; k < 3; ++k) dq0[j][1 + k] = m[k];
    }
    F hl[5], hr[5], Q0[5];
    half(ql, 1.0, hl);
    half(qr, -1.0, hr);
    for (int v = 0; v < 5; ++v) Q0[v] = hl[v] + hr[v];
    const ES es = estate(Q0);
    F dtQ[5] = {0, 0, 0, 0, 0}, jv[5];
    for (int j = 0; j < 3; ++j) { jvp(j, Q0, es, dq0[j], jv); for (int v = 0; v < 5; ++v) dtQ[v] -= jv[v]; }
    F dF[5], Fl[5];
    jvp(0, Q0, es, dtQ, dF);
    // stage 2 writes d_t F only: the Euler flux F and its rotation are stage-1 work
    const int s0 = stage == 1 ? 0 : 1;
    if (stage == 1) {
      F u = es.u[0];
      Fl[0] = Q0[1]; Fl[1] = Q0[1] * u + es.p; Fl[2] = Q0[2] * u; Fl[3] = Q0[3] * u; Fl[4] = u * es.H;
    }
    // back to the global frame, weighted, summed over the face
    F out[10];
    for (int s = s0; s < 2; ++s) {
      const F* A = s ? dF : Fl;
      out[5 * s] = wS * A[0];
      for (int a = 0; a < 3; ++a) out[5 * s + 1 + a] = wS * (A[1] * n[a] + A[2] * t1[a] + A[3] * t2[a]);
      out[5 * s + 4] = wS * A[4];
    }
    for (int k = 5 * s0; k < 10; ++k) sum[k] = g == 0 ? out[k] : sum[k] + out[k];
  }
  (void)face_part;
  return g_flops;
}
