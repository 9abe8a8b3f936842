// sm_100a fp64 kernels of the HGKS hot path.
//
//   k_bc_ghosts   a6  boundary-condition ghost states (wall mirror / farfield)
//   k_recon       a7  WENO reconstruction (tile-staged stencils): LSQ apply, beta, weights, collapse
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

// Conserved state of a cell: one 48-byte row (rho, rhoU, rhoV, rhoW, rhoE, pad),
// so a stencil gather is 3 aligned 16-byte loads and a ghost range is one
// contiguous block (single message per peer in the halo exchange).
constexpr int QS = 6;

// part 0: ghosts of owned cells (before the halo exchange completes), 1: ghosts
// of partition-ghost cells (after it), 2: all
__global__ void k_bc_ghosts(double* __restrict__ Q, int first, int n, const int* __restrict__ bg_cell,
                            const int* __restrict__ bg_bc, const double* __restrict__ bg_normal, GasParams gp,
                            int n_owned, int part) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (part != 2 && (bg_cell[k] < n_owned) != (part == 0)) return;
  const double* qc = Q + (size_t)bg_cell[k] * QS;
  double qi[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) qi[v] = qc[v];
  double qb[5];
  if (bg_bc[k] == 1) {
    qb[0] = qi[0]; qb[1] = -qi[1]; qb[2] = -qi[2]; qb[3] = -qi[3]; qb[4] = qi[4];
  } else {
    double n3[3] = {bg_normal[3 * k], bg_normal[3 * k + 1], bg_normal[3 * k + 2]};
    farfield_riemann(qi, n3, gp, qb);
  }
  double* qg = Q + (size_t)(first + k) * QS;
#pragma unroll
  for (int v = 0; v < 5; ++v) qg[v] = qb[v];
}

// ----------------------------------------------------------------------------
// a7: WENO reconstruction, one thread per reconstructed cell, 128-cell blocks.
// Output record per local cell (50 doubles), variable-major: for v = 0..4,
// rec[10 v + (const, x, y, z, xx, yy, zz, xy, xz, yz)] so that at X = x - c_i
//   Q_v(x) = const + lin . X + quad . (X_a X_b)       (Eq. weno collapsed)
// ----------------------------------------------------------------------------
constexpr int kRec = 50;
constexpr int kTile = 128;        // reconstructed cells per block

struct ReconArgs {
  const double* __restrict__ Q;         // [n_local][QS]
  int n_recon;
  int tile0;                            // first 128-cell tile of this launch
  int ld;                               // n_recon padded to kTile (tiled entry-major arrays, setup.cpp)
  const int* __restrict__ recon_cell;   // [n_recon] local cell id
  const int* __restrict__ st_id;        // [K] per cell, tiled: stencil member local ids
  const uint8_t* __restrict__ sub_slot; // [M*NM] per cell, tiled: sub-stencil member -> big-stencil slot
  const double* __restrict__ op;        // [E] per cell, tiled: LSQ operators in streaming order
  const double* __restrict__ geo;       // [8] per cell, tiled: V^{2/3}, V^{4/3}, M2 (xx,yy,zz,xy,xz,yz)
  double* __restrict__ ceff;            // [n_local][50]
  double eps;
  int omega_pow;
};

// One thread per reconstructed cell (block of kTile cells).  All stencil
// indices are loaded first and all member states are gathered at once into
// this thread's shared-memory slots (3 x 16-byte loads per member, ~40 loads in
// flight per thread), so the gathers cost one memory latency per cell; the
// sub-stencils re-read them from shared memory.  The LSQ operators (1584 B per
// tet cell, most of the kernel's HBM bytes) stream entry-major: each warp load
// is 256 contiguous bytes.
template <int K, int M, int NM>
#ifndef HGKS_RECON_MINB
#define HGKS_RECON_MINB 2
#endif
__global__ void __launch_bounds__(kTile, HGKS_RECON_MINB) k_recon(ReconArgs a) {
  constexpr int QP = 5 * kTile;                      // doubles per member plane: [v][thread]
  constexpr int E = 9 * K + 3 * M * NM;
  extern __shared__ __align__(16) double smem[];
  double* __restrict__ dqs = smem;                   // [K][5][kTile] Q_k - Q_i
  const int t = threadIdx.x;
  const int tile = a.tile0 + blockIdx.x;
  const int r = tile * kTile + t;
  int ci = r < a.n_recon ? __ldg(a.recon_cell + r) : -1;  // -1: padding
  const bool active = ci >= 0;
  if (!active) ci = 0;
  // tiled entry-major per-cell arrays (setup.cpp): entry e of this cell at (tile*NE + e)*kTile + t
  const size_t tb = (size_t)tile * kTile;
  const int* __restrict__ sid = a.st_id + tb * K + t;
  double qi[5];
  {
    const double2* q2 = reinterpret_cast<const double2*>(a.Q + (size_t)ci * QS);
    const double2 x0 = __ldg(q2), x1 = __ldg(q2 + 1), x2 = __ldg(q2 + 2);
    qi[0] = x0.x; qi[1] = x0.y; qi[2] = x1.x; qi[3] = x1.y; qi[4] = x2.x;
  }
#ifndef HGKS_NO_L2_PREFETCH
  // The block's operators are one contiguous E*kTile*8-byte range (tiled layout):
  // fire TMA bulk prefetches of it into L2 now, so the streamed operator loads
  // below see L2 rather than DRAM latency (the warps cannot keep enough loads
  // in flight at 255 registers).
  if (t < 8) {
    constexpr uint32_t bytes = (uint32_t)E * kTile * sizeof(double);
    constexpr uint32_t chunk = ((bytes / 8) + 15) / 16 * 16;
    const uint32_t off = t * chunk;
    if (off < bytes) {
      const uint32_t n = min(chunk, bytes - off);
      const char* src = reinterpret_cast<const char*>(a.op + tb * E) + off;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(n) : "memory");
    }
  }
#endif
  // gather the stencil members in groups (bounded registers, 7 x 3 loads in flight)
  constexpr int G = 7;
#pragma unroll
  for (int k0 = 0; k0 < K; k0 += G) {
    double2 x[G][3];
#pragma unroll
    for (int k = k0; k < k0 + G && k < K; ++k) {
      const double2* q2 = reinterpret_cast<const double2*>(a.Q + (size_t)__ldg(sid + k * kTile) * QS);
      x[k - k0][0] = __ldg(q2);
      x[k - k0][1] = __ldg(q2 + 1);
      x[k - k0][2] = __ldg(q2 + 2);
    }
#pragma unroll
    for (int k = k0; k < k0 + G && k < K; ++k) {
      double* d = dqs + k * QP + t;
      d[0 * kTile] = x[k - k0][0].x - qi[0];
      d[1 * kTile] = x[k - k0][0].y - qi[1];
      d[2 * kTile] = x[k - k0][1].x - qi[2];
      d[3 * kTile] = x[k - k0][1].y - qi[3];
      d[4 * kTile] = x[k - k0][2].x - qi[4];
    }
  }
  const double* __restrict__ op = a.op + tb * E + t;
  const double* __restrict__ geo = a.geo + tb * 8 + t;
  const uint8_t* __restrict__ ssl = a.sub_slot + tb * (M * NM) + t;
  const double V23 = __ldg(geo), V43 = __ldg(geo + kTile);
  double m2[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) m2[q] = __ldg(geo + (2 + q) * kTile);
  // ---- P_0: c[d][v] = sum_k A0+[d][k] (Q_k - Q_i)[v] ----
  double c[9][5];
#pragma unroll
  for (int d = 0; d < 9; ++d)
#pragma unroll
    for (int v = 0; v < 5; ++v) c[d][v] = 0.0;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    double dq[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) dq[v] = dqs[k * QP + v * kTile + t];
#pragma unroll
    for (int d = 0; d < 9; ++d) {
      const double w = __ldcs(op + (k * 9 + d) * kTile);
#pragma unroll
      for (int v = 0; v < 5; ++v) c[d][v] = fma(w, dq[v], c[d][v]);
    }
  }
  // smoothness indicator of P_0 (closed form SURVEY A.5)
  double beta0[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double gx[3] = {2.0 * c[3][v], c[6][v], c[7][v]}, gy[3] = {c[6][v], 2.0 * c[4][v], c[8][v]},
                 gz[3] = {c[7][v], c[8][v], 2.0 * c[5][v]};
    auto quadf = [&](const double g[3]) {
      return m2[0] * g[0] * g[0] + m2[1] * g[1] * g[1] + m2[2] * g[2] * g[2] +
             2.0 * (m2[3] * g[0] * g[1] + m2[4] * g[0] * g[2] + m2[5] * g[1] * g[2]);
    };
    const double s1 = c[0][v] * c[0][v] + c[1][v] * c[1][v] + c[2][v] * c[2][v] + quadf(gx) + quadf(gy) + quadf(gz);
    const double s2 = 4.0 * (c[3][v] * c[3][v] + c[4][v] * c[4][v] + c[5][v] * c[5][v]) + c[6][v] * c[6][v] +
                      c[7][v] * c[7][v] + c[8][v] * c[8][v];
    beta0[v] = V23 * s1 + V43 * s2;
  }
  const double* __restrict__ opm = op + (9 * K) * kTile;
  auto sub_slopes = [&](int m, double b[3][5]) {  // P_m over sub-stencil m
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int v = 0; v < 5; ++v) b[d][v] = 0.0;
#pragma unroll
    for (int j = 0; j < NM; ++j) {
      const int sl = __ldg(ssl + (m * NM + j) * kTile);
      double dq[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) dq[v] = dqs[sl * QP + v * kTile + t];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double w = __ldg(opm + ((m * NM + j) * 3 + d) * kTile);
#pragma unroll
        for (int v = 0; v < 5; ++v) b[d][v] = fma(w, dq[v], b[d][v]);
      }
    }
  };
  // ---- pass 1: beta_m and the nonlinear weights ----
  const double gm = 0.025, g0 = 1.0 - 0.025 * M;
  double al0[5], alm[M][5];
  {
    double tz[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double b[3][5];
      sub_slopes(m, b);
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        alm[m][v] = V23 * (b[0][v] * b[0][v] + b[1][v] * b[1][v] + b[2][v] * b[2][v]);  // beta_m
        tz[v] += fabs(beta0[v] - alm[m][v]);
      }
    }
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double tzv = tz[v] * (1.0 / M);
      const double r0 = tzv / (beta0[v] + a.eps);
      const double w0 = g0 * (1.0 + (a.omega_pow == 2 ? r0 * r0 : r0));
      double sum = w0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const double rm = tzv / (alm[m][v] + a.eps);
        alm[m][v] = gm * (1.0 + (a.omega_pow == 2 ? rm * rm : rm));  // omega_m
        sum += alm[m][v];
      }
      const double inv = 1.0 / sum;
      al0[v] = w0 * inv / g0;  // omega-bar_0 / gamma_0
#pragma unroll
      for (int m = 0; m < M; ++m) alm[m][v] = alm[m][v] * inv - al0[v] * gm;  // omega-bar_m - omega-bar_0 gamma_m/gamma_0
    }
  }
  // ---- collapse to one quadratic ----
  double lin[3][5];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int v = 0; v < 5; ++v) lin[d][v] = al0[v] * c[d][v];
#pragma unroll
  for (int m = 0; m < M; ++m) {  // pass 2: weighted sum of the sub-stencil slopes
    double b[3][5];
    sub_slopes(m, b);
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int v = 0; v < 5; ++v) lin[d][v] = fma(alm[m][v], b[d][v], lin[d][v]);
  }
  if (!active) return;
  double2* dst = reinterpret_cast<double2*>(a.ceff + (size_t)ci * kRec);
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    double quad[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) quad[q] = al0[v] * c[3 + q][v];
    // zero-mean basis: p_ab = X_a X_b - M2_ab
    const double cst = qi[v] - (quad[0] * m2[0] + quad[1] * m2[1] + quad[2] * m2[2] + quad[3] * m2[3] +
                                quad[4] * m2[4] + quad[5] * m2[5]);
    dst[5 * v + 0] = make_double2(cst, lin[0][v]);
    dst[5 * v + 1] = make_double2(lin[1][v], lin[2][v]);
    dst[5 * v + 2] = make_double2(quad[0], quad[1]);
    dst[5 * v + 3] = make_double2(quad[2], quad[3]);
    dst[5 * v + 4] = make_double2(quad[4], quad[5]);
  }
}

#include "flux.cuh"

// ----------------------------------------------------------------------------
// a10: L, d_t L and the S2O4 stages
// ----------------------------------------------------------------------------
struct UpdateArgs {
  double* __restrict__ Q;  // [n_local][QS]  (stage 1: Q^n -> Q*, stage 2: -> Q^{n+1})
  double* __restrict__ R;  // [n_owned][QS]
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
    const int e = __ldg(a.cf + p * a.n_owned + i);
    const int f = e >= 0 ? e : ~e;
    const double2* F = reinterpret_cast<const double2*>(a.F1 + (size_t)f * 10);
    double v10[10];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const double2 x = __ldg(F + k);
      v10[2 * k] = x.x;
      v10[2 * k + 1] = x.y;
    }
    if (e >= 0) {
#pragma unroll
      for (int v = 0; v < 5; ++v) { L[v] -= v10[v]; dL[v] -= v10[5 + v]; }
    } else {
#pragma unroll
      for (int v = 0; v < 5; ++v) { L[v] += v10[v]; dL[v] += v10[5 + v]; }
    }
  }
  const double iv = a.inv_v[i];
  const double dt = a.ctrl->dt;
  double* q = a.Q + (size_t)i * QS;
  double* r = a.R + (size_t)i * QS;
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double l = L[v] * iv, dl = dL[v] * iv;
    const double q0 = q[v];
    q[v] = q0 + 0.5 * dt * l + 0.125 * dt * dt * dl;
    r[v] = q0 + dt * l + dt * dt / 6.0 * dl;
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
      const int e = __ldg(a.cf + p * a.n_owned + i);
      const int f = e >= 0 ? e : ~e;
      const double* F = a.F2 + (size_t)f * 5;
      if (e >= 0) {
#pragma unroll
        for (int v = 0; v < 5; ++v) dL[v] -= __ldg(F + v);
      } else {
#pragma unroll
        for (int v = 0; v < 5; ++v) dL[v] += __ldg(F + v);
      }
    }
    const double iv = a.inv_v[i];
    const double dt = a.ctrl->dt;
    double q[5];
    const double* r = a.R + (size_t)i * QS;
    double* qo = a.Q + (size_t)i * QS;
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      q[v] = r[v] + dt * dt / 6.0 * 2.0 * (dL[v] * iv);
      qo[v] = q[v];
    }
    const double p = (a.gp.gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
    if (!(q[0] > 0.0) || !(p > 0.0)) atomicMin(&a.ctrl->bad_cell, i);
    else bound = cell_dt_bound(q, a.h_dt[i], a.gp);
  }
  block_min_dt(bound, a.ctrl);
}

__global__ void __launch_bounds__(256) k_dt_init(const double* __restrict__ Q, const double* __restrict__ h_dt, int n,
                                                 Ctrl* ctrl, GasParams gp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double bound = 1e300;
  if (i < n) {
    double q[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) q[v] = Q[(size_t)i * QS + v];
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

// state layout conversions for set/get_state: AoS [n][5] in caller order <-> local rows
__global__ void k_scatter_state(const double* __restrict__ in, const int64_t* __restrict__ row, int n,
                                double* __restrict__ Q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = row[i];
#pragma unroll
  for (int v = 0; v < 5; ++v) Q[(size_t)i * QS + v] = in[r * 5 + v];
  Q[(size_t)i * QS + 5] = 0.0;
}
__global__ void k_gather_state(const double* __restrict__ Q, const int* __restrict__ local_of_out, int n,
                               double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = local_of_out[k];
#pragma unroll
  for (int v = 0; v < 5; ++v) out[(size_t)k * 5 + v] = Q[(size_t)i * QS + v];
}
// halo pack: rows of the send list, [n_send][QS]
__global__ void k_pack(const double* __restrict__ Q, const int* __restrict__ list, int n, double* __restrict__ buf) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n * 3) return;
  const int j = k / 3, part = k - 3 * j;
  reinterpret_cast<double2*>(buf)[k] = reinterpret_cast<const double2*>(Q + (size_t)list[j] * QS)[part];
}

}  // namespace hgks
