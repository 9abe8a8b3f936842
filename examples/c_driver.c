/* Minimal C user of libhgks (no Python): a periodic box of N^3 hexahedra on
 * [0,2]^3 carrying a smooth density wave, advanced 20 S2O4 steps on the GPU
 * through the C-ABI of include/hgks.h.  Checks discrete conservation of mass
 * and energy (the update is a sum of face fluxes) and prints them.
 *
 *   gcc -std=c11 -O2 -Iinclude -I/usr/local/cuda/include examples/c_driver.c \
 *       -Lpaper_2407_00656_b200 -lhgks -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2407_00656_b200 -lm -o c_driver && ./c_driver 24
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hgks.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    hgks_status s_ = (x);                                                          \
    if (s_ != HGKS_OK) {                                                           \
      fprintf(stderr, "%s failed (%d): %s\n", #x, (int)s_, hgks_last_error());     \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 16;
  const int64_t nn = (int64_t)(N + 1) * (N + 1) * (N + 1), nc = (int64_t)N * N * N;
  const double h = 2.0 / N, gamma = 1.4, PI = 3.14159265358979323846;
  double* xyz = malloc(sizeof(double) * 3 * nn);
  int8_t* type = malloc(nc);
  int64_t* cells = malloc(sizeof(int64_t) * 8 * nc);
  double* Q = malloc(sizeof(double) * 5 * nc);
  double* Qout = malloc(sizeof(double) * 5 * nc);
#define NID(i, j, k) ((int64_t)(k) * (N + 1) * (N + 1) + (int64_t)(j) * (N + 1) + (i))
  for (int k = 0; k <= N; ++k)
    for (int j = 0; j <= N; ++j)
      for (int i = 0; i <= N; ++i) {
        double* p = xyz + 3 * NID(i, j, k);
        p[0] = i * h; p[1] = j * h; p[2] = k * h;
      }
  for (int k = 0; k < N; ++k)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) {
        const int64_t c = ((int64_t)k * N + j) * N + i;
        int64_t* v = cells + 8 * c;  /* VTK order: bottom 0-3, top 4-7 */
        v[0] = NID(i, j, k); v[1] = NID(i + 1, j, k); v[2] = NID(i + 1, j + 1, k); v[3] = NID(i, j + 1, k);
        v[4] = NID(i, j, k + 1); v[5] = NID(i + 1, j, k + 1); v[6] = NID(i + 1, j + 1, k + 1); v[7] = NID(i, j + 1, k + 1);
        type[c] = HGKS_HEX;
        const double x = (i + 0.5) * h, y = (j + 0.5) * h, z = (k + 0.5) * h;
        const double rho = 1.0 + 0.2 * sin(PI * (x + y + z)), p = 1.0;
        double* q = Q + 5 * c;
        q[0] = rho; q[1] = q[2] = q[3] = rho;  /* U = V = W = 1 */
        q[4] = p / (gamma - 1.0) + 1.5 * rho;
      }
  hgks_mesh_desc d = {0};
  d.xyz = xyz; d.n_nodes = nn; d.cell_type = type; d.cell_nodes = cells; d.n_cells = nc;
  for (int a = 0; a < 3; ++a) { d.periodic_origin[a] = 0.0; d.periodic_length[a] = 2.0; }
  d.n_ranks = 1;
  hgks_mesh* mesh = NULL;
  CHECK(hgks_mesh_create(&d, &mesh));
  hgks_config cfg = {0};
  cfg.gamma = gamma; cfg.cfl = 0.5; cfg.tau_mode = 0; cfg.c1 = 1.0; cfg.t_inf = 1.0; cfg.mu_exp = 0.7;
  cfg.eps = 1e-10; cfg.omega_pow = 1; cfg.precision = 64;
  cfg.freestream[0] = 1.0; cfg.freestream[4] = 1.0 / gamma;
  size_t bytes = 0;
  CHECK(hgks_workspace_size(mesh, &cfg, 0, &bytes));
  void* ws = NULL;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) { fprintf(stderr, "cudaMalloc failed\n"); return 1; }
  cudaStream_t st;
  cudaStreamCreate(&st);
  hgks_solver* s = NULL;
  CHECK(hgks_init(mesh, &cfg, NULL, ws, bytes, (void*)st, Q, &s));
  hgks_step_info info;
  CHECK(hgks_step(s, 20, 0.0, &info));
  double t = 0.0;
  CHECK(hgks_get_state(s, Qout, NULL, &t));
  double m0 = 0, m1 = 0, e0 = 0, e1 = 0;
  for (int64_t c = 0; c < nc; ++c) { m0 += Q[5 * c]; m1 += Qout[5 * c]; e0 += Q[5 * c + 4]; e1 += Qout[5 * c + 4]; }
  const double dm = fabs(m1 - m0) / m0, de = fabs(e1 - e0) / e0;
  printf("%s: %lld hexes, %lld steps, t = %.6f, dt = %.3e, mass drift %.2e, energy drift %.2e -> %s\n",
         hgks_version(), (long long)nc, (long long)info.steps_done, t, info.last_dt, dm, de,
         (dm < 1e-12 && de < 1e-12) ? "OK" : "FAIL");
  CHECK(hgks_destroy(s));
  CHECK(hgks_mesh_destroy(mesh));
  cudaFree(ws);
  cudaStreamDestroy(st);
  free(xyz); free(type); free(cells); free(Q); free(Qout);
  return (dm < 1e-12 && de < 1e-12) ? 0 : 2;
}
