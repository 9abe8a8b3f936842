// Precision-independent device code of libhgks: the step control block, the
// CFL bound and its exact min (fp64 in both precisions), the time bookkeeping.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "erfc_fit.h"

namespace hgks {

// erfc(z) together with exp(-z^2), which the half-range Maxwellian moments need both
// of.  fp64: erfcx(|z|) = P(t)/(|z| + K), t = (|z| - K)/(|z| + K), P a
// degree-22 polynomial in t (Chebyshev fit emitted in the monomial basis, evaluated as four
// interleaved Horner chains in t^4; scripts/fit_erfc.py; absolute error of erfc
// <= 2e-15, tests/test_erfc_fit.py), so one exp serves both and the branchy library erfc
// (about 160 instructions per call in the flux kernels' SASS) is gone.  fp32: library calls.
// exp(x) for x <= 0 (the Maxwellian tail exp(-z^2), exp(-dt/tau)): Cody-Waite
// reduction x = k ln2 + r, |r| <= ln2/2 (two-part ln2), degree-12 Taylor series (even and
// odd parts as two Horner chains in r^2), 2^k
// added to the exponent field; relative error <= 4e-16 on [-700, 0], 0 below -700
// (tests/test_exp_neg.py).  About half the instructions of the library exp, which
// also handles positive arguments, overflow and NaN.
#ifndef HGKS_POLY_SPLIT
#define HGKS_POLY_SPLIT 1  // 0: single Horner chains (round-2 baseline, for A/B builds)
#endif
// 1/j! for even j = 12, 10, ..., 0 and odd j = 11, 9, ..., 1 (exp_neg's two Horner chains)
__constant__ double kExpEven[7] = {2.08767569878680989792e-09, 2.75573192239858906526e-07,
                                   2.48015873015873015873e-05, 1.38888888888888888889e-03,
                                   4.16666666666666666667e-02, 0.5, 1.0};
__constant__ double kExpOdd[6] = {2.50521083854417187751e-08, 2.75573192239858906526e-06,
                                  1.98412698412698412698e-04, 8.33333333333333333333e-03,
                                  1.66666666666666666667e-01, 1.0};
__device__ __forceinline__ double exp_neg(double x) {
  const double xc = fmax(x, -708.0);
  const double k = rint(xc * 1.4426950408889634);
  const double r = fma(-k, 1.90821492927058770002e-10, fma(-k, 6.93147180369123816490e-01, xc));
#if HGKS_POLY_SPLIT
  // sum_{j<=12} r^j / j! as even + r * odd parts in r^2: two independent Horner chains of
  // depth 6 / 5 instead of one of depth 12 (the flux kernels stall on dependent DFMAs); the
  // coefficients come from the constant bank (LDCU.128, two per load) instead of two UMOVs
  // per literal
  const double r2 = r * r;
  double pe = kExpEven[0], po = kExpOdd[0];
#pragma unroll
  for (int j = 1; j < 6; ++j) {
    pe = fma(pe, r2, kExpEven[j]);
    po = fma(po, r2, kExpOdd[j]);
  }
  pe = fma(pe, r2, kExpEven[6]);
  const double p = fma(po, r, pe);
#else
  double p = 2.08767569878680989792e-09;  // 1/12!
  p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
#endif
  const int ki = (int)k;  // in [-1022, 0]
  const double v = __hiloint2double(__double2hiint(p) + ki * (1 << 20), __double2loint(p));
  return x < -700.0 ? 0.0 : v;
}
__device__ __forceinline__ float exp_neg(float x) { return expf(x); }

// 1/x for a positive normal x (densities, x + K, face areas): the MUFU reciprocal estimate
// refined by two Newton steps (relative error ~1e-16, not correctly rounded), without the
// IEEE division's special-case test and slow-path call (HGKS_FAST_RCP=0: plain division)
#ifndef HGKS_FAST_RCP
#define HGKS_FAST_RCP 1
#endif
__device__ __forceinline__ double rcp_pos(double x) {
#if HGKS_FAST_RCP
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
#else
  return 1.0 / x;
#endif
}
__device__ __forceinline__ float rcp_pos(float x) { return 1.0f / x; }
// 1/sqrt(x) for a positive normal x: MUFU estimate and two Newton steps y (3 - x y^2) / 2
__device__ __forceinline__ double rsqrt_pos(double x) {
#if HGKS_FAST_RCP
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
#else
  return rsqrt(x);
#endif
}
__device__ __forceinline__ float rsqrt_pos(float x) { return rsqrtf(x); }

// (coefficients in constant memory: the DFMA/DADD take them as c[][] operands, no
// per-coefficient register moves)
__constant__ double kErfcCoef[HGKS_ERFC_DEG + 1] = HGKS_ERFC_COEF;
// FAST: 1/(|z| + K) by rcp_pos (the tau = 0 interior kernel; measured slower in the moment form)
template <bool FAST = false>
__device__ __forceinline__ void erfc_exp(double z, double& erfc_z, double& ez2) {
  const double* c = kErfcCoef;
  const double a = fabs(z);
  const double r = FAST ? rcp_pos(a + HGKS_ERFC_K) : 1.0 / (a + HGKS_ERFC_K);
  const double t = (a - HGKS_ERFC_K) * r;
#if HGKS_POLY_SPLIT
  // P(t) = P0(s) + t P1(s) + t^2 P2(s) + t^3 P3(s), s = t^4, P_i(s) = sum_j c_{4j+i} s^j:
  // four independent Horner chains (depth 5) and a depth-3 combination instead of one
  // chain of depth 22 (3 extra multiplies)
  const double t2 = t * t, s4 = t2 * t2;
  double Pi[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    constexpr int D = HGKS_ERFC_DEG;
    const int top = D - ((D - i) % 4);  // highest degree k <= D with k = i (mod 4)
    Pi[i] = c[top];
#pragma unroll
    for (int k = top - 4; k >= 0; k -= 4) Pi[i] = fma(Pi[i], s4, c[k]);
  }
  const double P = fma(fma(fma(Pi[3], t, Pi[2]), t, Pi[1]), t, Pi[0]);
#else
  double P = c[HGKS_ERFC_DEG];
#pragma unroll
  for (int k = HGKS_ERFC_DEG - 1; k >= 0; --k) P = fma(P, t, c[k]);
#endif
  ez2 = exp_neg(-z * z);
  const double v = P * r * ez2;  // erfc(|z|)
  erfc_z = z >= 0.0 ? v : 2.0 - v;
}
template <bool FAST = false>
__device__ __forceinline__ void erfc_exp(float z, float& erfc_z, float& ez2) {
  erfc_z = erfcf(z);
  ez2 = expf(-z * z);
}

constexpr int QS = 6;      // values per cell row of Q (5 conserved + 1 pad for 16-byte pairs)
constexpr int kRec = 50;   // values per effective-polynomial record (10 coefficients x 5 variables)
constexpr int kTile = 128; // reconstructed cells per k_recon block (tiled arrays, setup.cpp)

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
  double pr_fac;  // 1/Pr - 1: heat-flux (Prandtl-number) correction of the energy flux (R29); 0 = none
};


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
// f3 cross-process halo put: per-rank flag words in the workspace, written by peers
// over NVLink (system-scope release stores), read with acquire loads.
// arrived[q] = last stage epoch whose ghost rows rank q has put into this rank;
// consumed[p] = last stage epoch whose ghost rows rank p (a receiver of this rank's
// puts) has finished reading.
struct P2PFlags {
  unsigned long long arrived[kMaxGroup];
  unsigned long long consumed[kMaxGroup];
  unsigned int put_blocks;  // blocks of the current k_put_release done (the last one releases)
  unsigned int pad[3];
};
struct P2PSignal {
  unsigned long long* dst[kMaxGroup];  // peer flag words (mapped peer memory)
  int n;
};
struct P2PWait {
  const unsigned long long* src[kMaxGroup];  // this rank's flag words
  int n;
};
// one thread: make this stream's earlier writes (the put kernel's peer stores) visible
// system-wide, then publish the epoch to every peer flag
__global__ void k_p2p_signal(P2PSignal s, unsigned long long epoch) {
  if (threadIdx.x != 0) return;
  asm volatile("fence.sc.sys;" ::: "memory");
  for (int k = 0; k < s.n; ++k) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(s.dst[k]), "l"(epoch) : "memory");
}
// one thread: spin until every flag has reached the epoch (acquire: the peer's puts
// made before its release are visible to the kernels that follow on this stream)
__global__ void k_p2p_wait(P2PWait w, unsigned long long epoch) {
  if (threadIdx.x != 0) return;
  for (int k = 0; k < w.n; ++k) {
    unsigned long long v;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(w.src[k]) : "memory");
      if (v < epoch) __nanosleep(200);
    } while (v < epoch);
  }
}

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


}  // namespace hgks
