// sm_100a fp64 kernels of the HGKS hot path.
//
//   k_bc_ghosts   a6  boundary-condition ghost states (wall mirror / farfield)
//   k_recon       a7  WENO reconstruction: LSQ apply, beta, weights, collapse
//                     to ONE effective quadratic per cell (50 doubles)
//   k_flux_tau0   a8+a9 per Gauss point: evaluate both polynomials, local
//                     frame, Q0 by kinetic upwinding, F and d_t F of f = g0(1+A t)
//                     via the Euler-chain identity, face quadrature sum
//   k_update1/2   a10 L, d_t L assembly in local-face order + S2O4 stages;
//                     stage 2 fuses the per-cell CFL bound and its min (a4)
//
// No tensor cores: there is no dense contraction on this path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hgks {

struct Ctrl {
  double t;          // time at the start of the current step
  double dt;         // step size of the current step
  double t_next;     // time after the current step
  unsigned long long dtmin_bits;  // min over cells of h/(|U|+c+2nu/h), as ordered bits
  long long steps;   // steps with dt > 0
  long long fallbacks;
  int bad_cell;      // first cell with non-positive rho/p (INT_MAX if none)
  int pad;
};

struct GasParams {
  double gamma, K, cfl, fixed_dt, eps, omega_pow;
  int tau_mode;
  double c1, mu_inf, t_inf, mu_exp;
  double fs[5];
};

// ----------------------------------------------------------------------------
// a6: boundary ghost states (R25).  Wall: velocity reversed.  Farfield: 1-D
// Riemann invariants along the face normal.
// ----------------------------------------------------------------------------
__device__ inline void farfield_riemann(const double qi[5], const double n[3], const GasParams& gp, double qb[5]) {
  const double g = gp.gamma;
  double rho_i = qi[0];
  double ui[3] = {qi[1] / rho_i, qi[2] / rho_i, qi[3] / rho_i};
  double p_i = (g - 1.0) * (qi[4] - 0.5 * (qi[1] * ui[0] + qi[2] * ui[1] + qi[3] * ui[2]));
  double c_i = sqrt(g * p_i / rho_i);
  double rho_f = gp.fs[0], p_f = gp.fs[4];
  double uf[3] = {gp.fs[1], gp.fs[2], gp.fs[3]};
  double c_f = sqrt(g * p_f / rho_f);
  double un_i = ui[0] * n[0] + ui[1] * n[1] + ui[2] * n[2];
  double un_f = uf[0] * n[0] + uf[1] * n[1] + uf[2] * n[2];
  double Rp = un_i + 2.0 * c_i / (g - 1.0), Rm = un_f - 2.0 * c_f / (g - 1.0);
  if (un_f + c_f < 0.0) Rp = un_f + 2.0 * c_f / (g - 1.0);
  if (un_i - c_i > 0.0) Rm = un_i - 2.0 * c_i / (g - 1.0);
  double un = 0.5 * (Rp + Rm), c = 0.25 * (g - 1.0) * (Rp - Rm);
  double ut[3], s;
  if (un > 0.0) {
    for (int a = 0; a < 3; ++a) ut[a] = ui[a] - un_i * n[a];
    s = p_i / pow(rho_i, g);
  } else {
    for (int a = 0; a < 3; ++a) ut[a] = uf[a] - un_f * n[a];
    s = p_f / pow(rho_f, g);
  }
  double rho = pow(c * c / (g * s), 1.0 / (g - 1.0));
  double p = rho * c * c / g;
  double u[3] = {ut[0] + un * n[0], ut[1] + un * n[1], ut[2] + un * n[2]};
  qb[0] = rho;
  qb[1] = rho * u[0];
  qb[2] = rho * u[1];
  qb[3] = rho * u[2];
  qb[4] = p / (g - 1.0) + 0.5 * rho * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
}

__global__ void k_bc_ghosts(double* __restrict__ Q, int ldq, int first, int n, const int* __restrict__ bg_cell,
                            const int* __restrict__ bg_bc, const double* __restrict__ bg_normal, GasParams gp) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int c = bg_cell[k];
  double qi[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) qi[v] = Q[v * ldq + c];
  double qb[5];
  if (bg_bc[k] == 1) {
    qb[0] = qi[0]; qb[1] = -qi[1]; qb[2] = -qi[2]; qb[3] = -qi[3]; qb[4] = qi[4];
  } else {
    double n3[3] = {bg_normal[3 * k], bg_normal[3 * k + 1], bg_normal[3 * k + 2]};
    farfield_riemann(qi, n3, gp, qb);
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) Q[v * ldq + first + k] = qb[v];
}

// ----------------------------------------------------------------------------
// a7: WENO reconstruction, one thread per reconstructed cell.
// Output record per local cell (50 doubles): [const(5) | lin x,y,z (3x5) |
// quad xx,yy,zz,xy,xz,yz (6x5)], so that at X = x - c_i
//   Q(x) = const + sum_a lin_a X_a + quad . (X_a X_b)       (Eq. weno collapsed)
// ----------------------------------------------------------------------------
constexpr int kRec = 50;

struct ReconArgs {
  const double* __restrict__ Q;  // [5][ldq]
  int ldq;
  int n_recon;
  const int* __restrict__ recon_cell;
  const int* __restrict__ st_id;        // [K][n_recon]
  const uint8_t* __restrict__ sub_slot; // [M*NM][n_recon]
  const double* __restrict__ op;        // [E][n_recon]
  const double* __restrict__ geo;       // [8][n_recon]
  double* __restrict__ ceff;            // [n_cells_local][50]
  double eps;
  int omega_pow;
};

// One thread per (cell, conserved variable): the smoothness indicators and the
// nonlinear weights are per variable (R12), so the five variables of a cell
// are independent.  Block = CT cells x 5 variables; warp y = variable y of CT
// consecutive cells, so every operator load is a coalesced 256-byte row read
// by 5 warps (one HBM fetch, L1 hits for the other four) and each thread keeps
// only 9 + 3M accumulators live (4x fewer registers -> 4x more warps in flight
// for the stencil gathers than one thread per cell).
template <int K, int M, int NM, int CT>
__global__ void __launch_bounds__(CT * 5) k_recon_v(ReconArgs a) {
  const int r = blockIdx.x * CT + threadIdx.x;
  const int v = threadIdx.y;
  if (r >= a.n_recon) return;
  const int R = a.n_recon;
  const int ci = __ldg(a.recon_cell + r);
  const double* __restrict__ Qv = a.Q + (size_t)v * a.ldq;
  const double qi = __ldg(Qv + ci);
  const double* __restrict__ op = a.op + r;
  // ---- P_0: c[d] = sum_k A0+[d][k] (Q_k - Q_i) ----
  double c[9];
#pragma unroll
  for (int d = 0; d < 9; ++d) c[d] = 0.0;
#pragma unroll 7
  for (int k = 0; k < K; ++k) {
    const double dq = __ldg(Qv + __ldg(a.st_id + k * R + r)) - qi;
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = fma(__ldg(op + (size_t)(d * K + k) * R), dq, c[d]);
  }
  // ---- P_m over the sub-stencils ----
  double b[M][3];
  const double* __restrict__ opm = op + (size_t)(9 * K) * R;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    b[m][0] = b[m][1] = b[m][2] = 0.0;
#pragma unroll
    for (int j = 0; j < NM; ++j) {
      const int s = __ldg(a.sub_slot + (m * NM + j) * R + r);
      const double dq = __ldg(Qv + __ldg(a.st_id + s * R + r)) - qi;
#pragma unroll
      for (int d = 0; d < 3; ++d) b[m][d] = fma(__ldg(opm + (size_t)((m * 3 + d) * NM + j) * R), dq, b[m][d]);
    }
  }
  const double V23 = __ldg(a.geo + r), V43 = __ldg(a.geo + R + r);
  double m2[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) m2[q] = __ldg(a.geo + (2 + q) * R + r);
  // ---- smoothness indicators (closed form SURVEY A.5) ----
  double beta0;
  {
    const double gx[3] = {2.0 * c[3], c[6], c[7]}, gy[3] = {c[6], 2.0 * c[4], c[8]}, gz[3] = {c[7], c[8], 2.0 * c[5]};
    auto quadf = [&](const double g[3]) {
      return m2[0] * g[0] * g[0] + m2[1] * g[1] * g[1] + m2[2] * g[2] * g[2] +
             2.0 * (m2[3] * g[0] * g[1] + m2[4] * g[0] * g[2] + m2[5] * g[1] * g[2]);
    };
    const double s1 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2] + quadf(gx) + quadf(gy) + quadf(gz);
    const double s2 = 4.0 * (c[3] * c[3] + c[4] * c[4] + c[5] * c[5]) + c[6] * c[6] + c[7] * c[7] + c[8] * c[8];
    beta0 = V23 * s1 + V43 * s2;
  }
  double betam[M];
#pragma unroll
  for (int m = 0; m < M; ++m) betam[m] = V23 * (b[m][0] * b[m][0] + b[m][1] * b[m][1] + b[m][2] * b[m][2]);
  // ---- nonlinear weights and the collapse ----
  const double gm = 0.025, g0 = 1.0 - 0.025 * M;
  double tz = 0.0;
#pragma unroll
  for (int m = 0; m < M; ++m) tz += fabs(beta0 - betam[m]);
  tz *= (1.0 / M);
  const double r0 = tz / (beta0 + a.eps);
  const double w0 = g0 * (1.0 + (a.omega_pow == 2 ? r0 * r0 : r0));
  double wm[M], sum = w0;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double rm = tz / (betam[m] + a.eps);
    wm[m] = gm * (1.0 + (a.omega_pow == 2 ? rm * rm : rm));
    sum += wm[m];
  }
  const double inv = 1.0 / sum;
  const double al0 = w0 * inv / g0;  // omega-bar_0 / gamma_0
  double lin[3] = {al0 * c[0], al0 * c[1], al0 * c[2]};
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double alm = wm[m] * inv - al0 * gm;  // omega-bar_m - omega-bar_0 gamma_m / gamma_0
#pragma unroll
    for (int d = 0; d < 3; ++d) lin[d] = fma(alm, b[m][d], lin[d]);
  }
  double quad[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) quad[q] = al0 * c[3 + q];
  const double cst = qi - (quad[0] * m2[0] + quad[1] * m2[1] + quad[2] * m2[2] + quad[3] * m2[3] + quad[4] * m2[4] +
                           quad[5] * m2[5]);
  double* __restrict__ out = a.ceff + (size_t)ci * kRec;
  out[v] = cst;
#pragma unroll
  for (int d = 0; d < 3; ++d) out[5 + d * 5 + v] = lin[d];
#pragma unroll
  for (int q = 0; q < 6; ++q) out[20 + q * 5 + v] = quad[q];
}

template <int K, int M, int NM, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_recon(ReconArgs a) {
  extern __shared__ double sb[];  // [M*15][BLOCK] sub-stencil slopes
  const int r = blockIdx.x * BLOCK + threadIdx.x;
  if (r >= a.n_recon) return;
  const int R = a.n_recon;
  const int ci = a.recon_cell[r];
  const double* __restrict__ Q = a.Q;
  const int ldq = a.ldq;
  double qi[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) qi[v] = Q[v * ldq + ci];
  // ---- P_0: c[d][v] = sum_k A0+[d][k] (Q_k - Q_i)[v] ----
  double c[9][5];
#pragma unroll
  for (int d = 0; d < 9; ++d)
#pragma unroll
    for (int v = 0; v < 5; ++v) c[d][v] = 0.0;
  const double* __restrict__ op = a.op + r;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    const int id = a.st_id[k * R + r];
    double dq[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) dq[v] = __ldg(Q + v * ldq + id) - qi[v];
#pragma unroll
    for (int d = 0; d < 9; ++d) {
      const double w = __ldcs(op + (size_t)(d * K + k) * R);
#pragma unroll
      for (int v = 0; v < 5; ++v) c[d][v] = fma(w, dq[v], c[d][v]);
    }
  }
  const double V23 = a.geo[0 * R + r], V43 = a.geo[1 * R + r];
  double m2[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) m2[q] = a.geo[(2 + q) * R + r];
  // ---- beta_0 closed form ----
  double beta0[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double cx = c[0][v], cy = c[1][v], cz = c[2][v];
    const double cxx = c[3][v], cyy = c[4][v], czz = c[5][v], cxy = c[6][v], cxz = c[7][v], cyz = c[8][v];
    // gradient d_a P0 = c_a + g_a . X ; g_x = (2cxx, cxy, cxz) ...
    const double gx[3] = {2.0 * cxx, cxy, cxz}, gy[3] = {cxy, 2.0 * cyy, cyz}, gz[3] = {cxz, cyz, 2.0 * czz};
    auto quadf = [&](const double g[3]) {
      return m2[0] * g[0] * g[0] + m2[1] * g[1] * g[1] + m2[2] * g[2] * g[2] +
             2.0 * (m2[3] * g[0] * g[1] + m2[4] * g[0] * g[2] + m2[5] * g[1] * g[2]);
    };
    const double s1 = cx * cx + cy * cy + cz * cz + quadf(gx) + quadf(gy) + quadf(gz);
    const double s2 = 4.0 * (cxx * cxx + cyy * cyy + czz * czz) + cxy * cxy + cxz * cxz + cyz * cyz;
    beta0[v] = V23 * s1 + V43 * s2;
  }
  // ---- P_m: b[d][v] over the sub-stencils, beta_m ----
  double betam[M][5];
  const double* __restrict__ opm = op + (size_t)(9 * K) * R;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    double b[3][5];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int v = 0; v < 5; ++v) b[d][v] = 0.0;
#pragma unroll
    for (int j = 0; j < NM; ++j) {
      const int s = a.sub_slot[(m * NM + j) * R + r];
      const int id = a.st_id[s * R + r];
      double dq[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) dq[v] = __ldg(Q + v * ldq + id) - qi[v];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double w = __ldcs(opm + (size_t)((m * 3 + d) * NM + j) * R);
#pragma unroll
        for (int v = 0; v < 5; ++v) b[d][v] = fma(w, dq[v], b[d][v]);
      }
    }
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      betam[m][v] = V23 * (b[0][v] * b[0][v] + b[1][v] * b[1][v] + b[2][v] * b[2][v]);
#pragma unroll
      for (int d = 0; d < 3; ++d) sb[((m * 3 + d) * 5 + v) * BLOCK + threadIdx.x] = b[d][v];
    }
  }
  // ---- nonlinear weights and collapse ----
  const double gm = 0.025, g0 = 1.0 - 0.025 * M;
  double* __restrict__ out = a.ceff + (size_t)ci * kRec;
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    double tz = 0.0;
#pragma unroll
    for (int m = 0; m < M; ++m) tz += fabs(beta0[v] - betam[m][v]);
    tz *= (1.0 / M);
    double r0 = tz / (beta0[v] + a.eps);
    double w0 = g0 * (1.0 + (a.omega_pow == 2 ? r0 * r0 : r0));
    double wm[M], sum = w0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double rm = tz / (betam[m][v] + a.eps);
      wm[m] = gm * (1.0 + (a.omega_pow == 2 ? rm * rm : rm));
      sum += wm[m];
    }
    const double inv = 1.0 / sum;
    const double al0 = w0 * inv / g0;  // omega-bar_0 / gamma_0
    double lin[3] = {al0 * c[0][v], al0 * c[1][v], al0 * c[2][v]};
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double alm = wm[m] * inv - al0 * gm;  // omega-bar_m - omega-bar_0 gamma_m / gamma_0
#pragma unroll
      for (int d = 0; d < 3; ++d) lin[d] = fma(alm, sb[((m * 3 + d) * 5 + v) * BLOCK + threadIdx.x], lin[d]);
    }
    double quad[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) quad[q] = al0 * c[3 + q][v];
    double cst = qi[v] - (quad[0] * m2[0] + quad[1] * m2[1] + quad[2] * m2[2] + quad[3] * m2[3] + quad[4] * m2[4] +
                          quad[5] * m2[5]);
    out[v] = cst;
#pragma unroll
    for (int d = 0; d < 3; ++d) out[5 + d * 5 + v] = lin[d];
#pragma unroll
    for (int q = 0; q < 6; ++q) out[20 + q * 5 + v] = quad[q];
  }
}

#include "flux.cuh"

// ----------------------------------------------------------------------------
// a10: L, d_t L and the S2O4 stages
// ----------------------------------------------------------------------------
struct UpdateArgs {
  double* __restrict__ Q;  // [5][ldq]  (stage 1: Q^n -> Q*, stage 2: -> Q^{n+1})
  int ldq;
  double* __restrict__ R;  // [5][n_owned]
  const double* __restrict__ F1;
  const double* __restrict__ F2;
  const int* __restrict__ cf;  // [NF][n_owned]
  const double* __restrict__ inv_v;
  const double* __restrict__ h_dt;
  int n_owned;
  Ctrl* ctrl;
  GasParams gp;
};

template <int NF>
__global__ void __launch_bounds__(256) k_update1(UpdateArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_owned) return;
  double L[5] = {0, 0, 0, 0, 0}, dL[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int p = 0; p < NF; ++p) {  // local-face order (deterministic, partition independent)
    const int e = a.cf[p * a.n_owned + i];
    const int f = e >= 0 ? e : ~e;
    const double* F = a.F1 + (size_t)f * 10;
    if (e >= 0) {
#pragma unroll
      for (int v = 0; v < 5; ++v) { L[v] -= F[v]; dL[v] -= F[5 + v]; }
    } else {
#pragma unroll
      for (int v = 0; v < 5; ++v) { L[v] += F[v]; dL[v] += F[5 + v]; }
    }
  }
  const double iv = a.inv_v[i];
  const double dt = a.ctrl->dt;
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double l = L[v] * iv, dl = dL[v] * iv;
    const double q = a.Q[v * a.ldq + i];
    a.Q[v * a.ldq + i] = q + 0.5 * dt * l + 0.125 * dt * dt * dl;
    a.R[v * a.n_owned + i] = q + dt * l + dt * dt / 6.0 * dl;
  }
}

__device__ __forceinline__ double cell_dt_bound(const double q[5], double h, const GasParams& gp) {
  const double rho = q[0];
  const double u = q[1] / rho, v = q[2] / rho, w = q[3] / rho;
  const double p = (gp.gamma - 1.0) * (q[4] - 0.5 * rho * (u * u + v * v + w * w));
  const double c = sqrt(gp.gamma * p / rho);
  double nu = 0.0;
  if (gp.tau_mode == 1) nu = gp.mu_inf * pow((p / rho) / gp.t_inf, gp.mu_exp) / rho;
  return h / (sqrt(u * u + v * v + w * w) + c + 2.0 * nu / h);
}

__device__ __forceinline__ void block_min_dt(double local, Ctrl* ctrl) {
  // warp shuffle min, then one atomic per warp on the ordered bits of a positive double
  unsigned long long bits = __double_as_longlong(local);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = ob < bits ? ob : bits;
  }
  if ((threadIdx.x & 31) == 0) atomicMin(&ctrl->dtmin_bits, bits);
}

template <int NF>
__global__ void __launch_bounds__(256) k_update2(UpdateArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double bound = 1e300;
  if (i < a.n_owned) {
    double dL[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int p = 0; p < NF; ++p) {
      const int e = a.cf[p * a.n_owned + i];
      const int f = e >= 0 ? e : ~e;
      const double* F = a.F2 + (size_t)f * 5;
      if (e >= 0) {
#pragma unroll
        for (int v = 0; v < 5; ++v) dL[v] -= F[v];
      } else {
#pragma unroll
        for (int v = 0; v < 5; ++v) dL[v] += F[v];
      }
    }
    const double iv = a.inv_v[i];
    const double dt = a.ctrl->dt;
    double q[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      q[v] = a.R[v * a.n_owned + i] + dt * dt / 6.0 * 2.0 * (dL[v] * iv);
      a.Q[v * a.ldq + i] = q[v];
    }
    const double p = (a.gp.gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
    if (!(q[0] > 0.0) || !(p > 0.0)) atomicMin(&a.ctrl->bad_cell, i);
    else bound = cell_dt_bound(q, a.h_dt[i], a.gp);
  }
  block_min_dt(bound, a.ctrl);
}

__global__ void __launch_bounds__(256) k_dt_init(const double* __restrict__ Q, int ldq, const double* __restrict__ h_dt,
                                                 int n, Ctrl* ctrl, GasParams gp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double bound = 1e300;
  if (i < n) {
    double q[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) q[v] = Q[v * ldq + i];
    bound = cell_dt_bound(q, h_dt[i], gp);
  }
  block_min_dt(bound, ctrl);
}

// one thread: advance the time bookkeeping and choose this step's dt
__global__ void k_step_begin(Ctrl* ctrl, double cfl, double fixed_dt, double t_stop) {
  double t = ctrl->t_next;
  double raw = fixed_dt > 0.0 ? fixed_dt : cfl * __longlong_as_double((long long)ctrl->dtmin_bits);
  double dt = raw, tn = t + raw;
  if (t_stop > 0.0) {
    if (t >= t_stop) {
      dt = 0.0;
      tn = t;
    } else if (t + raw > t_stop) {
      dt = t_stop - t;
      tn = t_stop;
    }
  }
  ctrl->t = t;
  ctrl->dt = dt;
  ctrl->t_next = tn;
  if (dt > 0.0) ctrl->steps += 1;
  ctrl->dtmin_bits = 0x7fefffffffffffffull;  // +max finite, reset for this step's accumulation
}

// loopback transport: exact min of the CFL bound over the ranks of one process
constexpr int kMaxGroup = 16;
struct GroupCtrl {
  int n;
  Ctrl* c[kMaxGroup];
};
__global__ void k_group_min(GroupCtrl g) {
  if (threadIdx.x != 0) return;
  unsigned long long m = g.c[0]->dtmin_bits;
  for (int k = 1; k < g.n; ++k) m = g.c[k]->dtmin_bits < m ? g.c[k]->dtmin_bits : m;
  for (int k = 0; k < g.n; ++k) g.c[k]->dtmin_bits = m;
}

// reset the time bookkeeping on the device (no host round trip)
__global__ void k_reset_ctrl(Ctrl* ctrl, double t) {
  ctrl->t = t;
  ctrl->t_next = t;
  ctrl->dt = 0.0;
  ctrl->bad_cell = 0x7fffffff;
  ctrl->dtmin_bits = 0x7fefffffffffffffull;
}

// state layout conversions for set/get_state: AoS [n][5] in caller order <-> SoA local
__global__ void k_scatter_state(const double* __restrict__ in, const int64_t* __restrict__ row, int n,
                                double* __restrict__ Q, int ldq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = row[i];
#pragma unroll
  for (int v = 0; v < 5; ++v) Q[v * ldq + i] = in[r * 5 + v];
}
__global__ void k_gather_state(const double* __restrict__ Q, int ldq, const int* __restrict__ local_of_out, int n,
                               double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = local_of_out[k];
#pragma unroll
  for (int v = 0; v < 5; ++v) out[(size_t)k * 5 + v] = Q[v * ldq + i];
}
// halo pack: SoA send buffer [5][n_send]
__global__ void k_pack(const double* __restrict__ Q, int ldq, const int* __restrict__ list, int n,
                       double* __restrict__ buf) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = list[k];
#pragma unroll
  for (int v = 0; v < 5; ++v) buf[v * n + k] = Q[v * ldq + i];
}

}  // namespace hgks
