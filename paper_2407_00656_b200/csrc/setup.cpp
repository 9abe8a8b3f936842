// Host setup of libhgks: geometry, faces, periodic
// pairing, Alg. 1 stencils, least-squares operators, k-way partition with 3
// ghost layers, Morton renumbering.  Runs once per mesh; never on the hot path.
//
// Independent of oracle/ (shares no code): faces are matched by bucketing on
// the smallest node id, periodic faces by sorted canonical keys, least squares
// by Gram-Schmidt QR with re-orthogonalisation to an explicit pseudo-inverse.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <tuple>
#include <unordered_map>

#include "internal.h"

namespace hgks {
namespace {

// HGKS_SETUP_TIMING=1: phase times of the host setup on stderr
struct PhaseTimer {
  bool on = std::getenv("HGKS_SETUP_TIMING") != nullptr;
  const char* who;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit PhaseTimer(const char* w) : who(w) {}
  void lap(const char* phase) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hgks setup] %s: %-28s %8.3f s\n", who, phase,
                 std::chrono::duration<double>(t - t0).count());
    t0 = t;
  }
};

struct P3 {
  double x, y, z;
};
inline P3 operator+(P3 a, P3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline P3 operator-(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline P3 operator*(double s, P3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dotp(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline P3 crossp(P3 a, P3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double len(P3 a) { return std::sqrt(dotp(a, a)); }

// tet face p = nodes other than p; hex faces, VTK order (R17); prism (wedge)
// faces: the two triangles, then the three sides, VTK order (R30)
const int kTetF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
const int kHexF[6][4] = {{0, 1, 2, 3}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}, {4, 5, 6, 7}};
const int kPriF[5][4] = {{0, 1, 2, -1}, {3, 4, 5, -1}, {0, 1, 4, 3}, {1, 2, 5, 4}, {2, 0, 3, 5}};

// cell kinds are coded by their node count: 4 tet, 6 prism, 8 hex
inline int cell_nfaces(int t) { return t == 4 ? 4 : (t == 6 ? 5 : 6); }
// node slots of face p of a cell of kind t; returns the face's vertex count
inline int face_slots(int t, int p, int s[4]) {
  if (t == 4) {
    for (int q = 0; q < 3; ++q) s[q] = kTetF[p][q];
    return 3;
  }
  const int* f = t == 6 ? kPriF[p] : kHexF[p];
  for (int q = 0; q < 4; ++q) s[q] = f[q];
  return (t == 6 && p < 2) ? 3 : 4;
}

// --- cell geometry (a0) ------------------------------------------------------
void tet_geometry(const P3 v[4], double& V, P3& c, double m2[6]) {
  P3 a = v[1] - v[0], b = v[2] - v[0], d = v[3] - v[0];
  V = std::fabs(dotp(a, crossp(b, d))) / 6.0;
  c = 0.25 * (((v[0] + v[1]) + v[2]) + v[3]);
  for (int k = 0; k < 6; ++k) m2[k] = 0;
  for (int k = 0; k < 4; ++k) {
    P3 e = v[k] - c;
    m2[0] += e.x * e.x; m2[1] += e.y * e.y; m2[2] += e.z * e.z;
    m2[3] += e.x * e.y; m2[4] += e.x * e.z; m2[5] += e.y * e.z;
  }
  for (int k = 0; k < 6; ++k) m2[k] *= 0.05;  // mean of (x-c)(x-c)^T over a tet = (1/20) sum_k e_k e_k^T
}

void hex_geometry(const P3 v[8], double& V, P3& c, double m2[6]) {
  // trilinear map on [0,1]^3, tensor 3-point Gauss (exact for these integrands)
  const double s = std::sqrt(0.15);
  const double gx[3] = {0.5 - s, 0.5, 0.5 + s}, gw[3] = {5.0 / 18.0, 4.0 / 9.0, 5.0 / 18.0};
  P3 X[27];
  double W[27];
  int q = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k, ++q) {
        double r = gx[i], t = gx[j], u = gx[k];
        double Nr[2] = {1 - r, r}, Nt[2] = {1 - t, t}, Nu[2] = {1 - u, u};
        // VTK corner (a,b,c) offsets
        const int off[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
        P3 x{0, 0, 0}, dr{0, 0, 0}, dt{0, 0, 0}, du{0, 0, 0};
        for (int n = 0; n < 8; ++n) {
          int a = off[n][0], b = off[n][1], cc = off[n][2];
          double sa = a ? 1.0 : -1.0, sb = b ? 1.0 : -1.0, sc = cc ? 1.0 : -1.0;
          x = x + (Nr[a] * Nt[b] * Nu[cc]) * v[n];
          dr = dr + (sa * Nt[b] * Nu[cc]) * v[n];
          dt = dt + (Nr[a] * sb * Nu[cc]) * v[n];
          du = du + (Nr[a] * Nt[b] * sc) * v[n];
        }
        X[q] = x;
        W[q] = gw[i] * gw[j] * gw[k] * std::fabs(dotp(dr, crossp(dt, du)));
      }
  V = 0;
  P3 acc{0, 0, 0};
  for (int k = 0; k < 27; ++k) {
    V += W[k];
    acc = acc + W[k] * X[k];
  }
  c = (1.0 / V) * acc;
  for (int k = 0; k < 6; ++k) m2[k] = 0;
  for (int k = 0; k < 27; ++k) {
    P3 e = X[k] - c;
    double w = W[k] / V;
    m2[0] += w * e.x * e.x; m2[1] += w * e.y * e.y; m2[2] += w * e.z * e.z;
    m2[3] += w * e.x * e.y; m2[4] += w * e.x * e.z; m2[5] += w * e.y * e.z;
  }
}

// Wedge map x = sum_a lam_a(r, s) ((1 - u) v_a + u v_{a+3}), lam = (1 - r - s, r, s): the
// Jacobian is linear in (r, s) and quadratic in u, so V, the centroid and M2 need a rule exact
// to degree 3 in (r, s) and 4 in u.  The triangle is collapsed from the unit square
// (r = X, s = Y (1 - X), dr ds = (1 - X) dX dY: degree <= 4 in X, 3 in Y), so 3-point Gauss in
// X, Y and u is exact.
void prism_geometry(const P3 v[6], double& V, P3& c, double m2[6]) {
  const double s = std::sqrt(0.15);
  const double gx[3] = {0.5 - s, 0.5, 0.5 + s}, gw[3] = {5.0 / 18.0, 4.0 / 9.0, 5.0 / 18.0};
  P3 X[27];
  double W[27];
  int q = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k, ++q) {
        const double r = gx[i], t = gx[j] * (1.0 - gx[i]), u = gx[k];
        const double lam[3] = {1.0 - r - t, r, t};
        P3 x{0, 0, 0}, du{0, 0, 0};
        for (int a = 0; a < 3; ++a) {
          x = x + lam[a] * ((1.0 - u) * v[a] + u * v[a + 3]);
          du = du + lam[a] * (v[a + 3] - v[a]);
        }
        // d/dr and d/ds of the map: dlam/dr = (-1, 1, 0), dlam/ds = (-1, 0, 1)
        const P3 b0 = (1.0 - u) * v[0] + u * v[3], b1 = (1.0 - u) * v[1] + u * v[4], b2 = (1.0 - u) * v[2] + u * v[5];
        const P3 dr = b1 - b0, ds = b2 - b0;
        X[q] = x;
        W[q] = gw[i] * gw[j] * gw[k] * (1.0 - gx[i]) * std::fabs(dotp(dr, crossp(ds, du)));
      }
  V = 0;
  P3 acc{0, 0, 0};
  for (int k = 0; k < 27; ++k) {
    V += W[k];
    acc = acc + W[k] * X[k];
  }
  c = (1.0 / V) * acc;
  for (int k = 0; k < 6; ++k) m2[k] = 0;
  for (int k = 0; k < 27; ++k) {
    P3 e = X[k] - c;
    double w = W[k] / V;
    m2[0] += w * e.x * e.x; m2[1] += w * e.y * e.y; m2[2] += w * e.z * e.z;
    m2[3] += w * e.x * e.y; m2[4] += w * e.x * e.z; m2[5] += w * e.y * e.z;
  }
}

void cell_geometry(int t, const P3* v, double& V, P3& c, double m2[6]) {
  if (t == 4) tet_geometry(v, V, c, m2);
  else if (t == 6) prism_geometry(v, V, c, m2);
  else hex_geometry(v, V, c, m2);
}

// Face Gauss points (R10): positions, unit normals along the vertex order's
// right-hand rule, and weight*area.
int face_gps(int nv, const P3* p, P3* x, P3* n, double* wS) {
  if (nv == 3) {
    P3 nn = crossp(p[1] - p[0], p[2] - p[0]);
    double a2 = len(nn);
    for (int g = 0; g < 3; ++g) {
      double l[3] = {1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0};
      l[g] = 2.0 / 3.0;
      x[g] = (l[0] * p[0] + l[1] * p[1]) + l[2] * p[2];
      n[g] = (1.0 / a2) * nn;
      wS[g] = a2 / 6.0;
    }
    return 3;
  }
  const double h = 0.5 / std::sqrt(3.0);
  const double q[2] = {0.5 - h, 0.5 + h};
  for (int g = 0; g < 4; ++g) {
    double s = q[g & 1], t = q[g >> 1];
    x[g] = ((1 - s) * (1 - t)) * p[0] + (s * (1 - t)) * p[1] + (s * t) * p[2] + ((1 - s) * t) * p[3];
    P3 ds = (1 - t) * (p[1] - p[0]) + t * (p[2] - p[3]);
    P3 dt = (1 - s) * (p[3] - p[0]) + s * (p[2] - p[1]);
    P3 nn = crossp(ds, dt);
    double a = len(nn);
    n[g] = (1.0 / a) * nn;
    wS[g] = 0.25 * a;
  }
  return 4;
}

// --- least squares (a2): pseudo-inverse by Gram-Schmidt QR (CGS2) ----------
// A is m x n (row-major), returns P (n x m) with P A = I, least-squares sense.
bool pinv_qr(int m, int n, const double* A, double* P) {
  constexpr int kMaxM = 64, kMaxN = 9;  // stencils have <= 40 members, <= 9 unknowns
  if (m > kMaxM || n > kMaxN) return false;
  double Q[kMaxM * kMaxN], R[kMaxN * kMaxN];
  for (int k = 0; k < n * n; ++k) R[k] = 0.0;
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) Q[i * n + j] = A[i * n + j];
    for (int pass = 0; pass < 2; ++pass)
      for (int k = 0; k < j; ++k) {
        double r = 0;
        for (int i = 0; i < m; ++i) r += Q[i * n + k] * Q[i * n + j];
        R[k * n + j] += r;
        for (int i = 0; i < m; ++i) Q[i * n + j] -= r * Q[i * n + k];
      }
    double nr = 0, na = 0;
    for (int i = 0; i < m; ++i) {
      nr += Q[i * n + j] * Q[i * n + j];
      na += A[i * n + j] * A[i * n + j];
    }
    nr = std::sqrt(nr);
    if (!(nr > 1e-10 * std::sqrt(na)) || na == 0.0) return false;
    R[j * n + j] = nr;
    for (int i = 0; i < m; ++i) Q[i * n + j] /= nr;
  }
  // P = R^{-1} Q^T : back substitution per column of Q^T
  for (int i = 0; i < m; ++i)
    for (int r = n - 1; r >= 0; --r) {
      double s = Q[i * n + r];
      for (int k = r + 1; k < n; ++k) s -= R[r * n + k] * P[k * m + i];
      P[r * m + i] = s / R[r * n + r];
    }
  return true;
}

struct Member {
  int64_t id;
  P3 s;
};

inline bool same_shift(P3 a, P3 b) { return std::fabs(a.x - b.x) + std::fabs(a.y - b.y) + std::fabs(a.z - b.z) < 1e-9; }

// Morton key of a point in [lo, hi]^3 (21 bits per axis)
uint64_t spread21(uint64_t v) {
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

}  // namespace

// Boundary refinement of a k-way partition on the face-adjacency (dual) graph (P:730-739:
// balanced parts, few cut faces): Fiduccia-Mattheyses passes.  Each pass repeatedly moves the
// unlocked boundary cell with the largest gain (cut faces removed minus added when it joins
// the neighbouring part it shares most faces with), negative gains included, keeping every
// part within 0.5 % of the mean size; each cell moves at most once per pass, and the pass is
// rolled back to its best prefix.  Deterministic (ties by cell id, then lower rank).  The
// solution does not depend on the partition (bitwise equal for any partition),
// only the halo volume does.
static void refine_partition(GlobalMesh& gm, int nfc) {
  const int64_t nc = gm.nc;
  const int nr = gm.n_ranks;
  std::vector<int64_t> size(nr, 0);
  for (int64_t i = 0; i < nc; ++i) ++size[gm.part[i]];
  const double mean = (double)nc / nr;
  // every part within 0.5 % of the mean, so the largest and smallest differ by <= 1 %
  const int64_t hi = std::max((int64_t)std::floor(mean * 1.005), (int64_t)std::ceil(mean)),
                lo = std::min((int64_t)std::ceil(mean * 0.995), (int64_t)std::floor(mean));
  // best move of cell i: (gain, target part); target -1 if i is not on a part boundary
  auto best_move = [&](int64_t i, int& target) {
    const int p = gm.part[i];
    int own = 0, nb_part[6], nb_cnt[6], nn = 0;
    for (int q = 0; q < nfc; ++q) {
      const int64_t j = gm.nbr_id[i * 6 + q];
      if (j < 0 || j >= nc) continue;  // boundary ghost, or no face q (a tet of a hybrid mesh)
      const int r = gm.part[j];
      if (r == p) { ++own; continue; }
      int k = 0;
      while (k < nn && nb_part[k] != r) ++k;
      if (k == nn) { nb_part[nn] = r; nb_cnt[nn++] = 0; }
      ++nb_cnt[k];
    }
    target = -1;
    int best = -1;
    for (int k = 0; k < nn; ++k)
      if (nb_cnt[k] > best || (nb_cnt[k] == best && nb_part[k] < target)) { best = nb_cnt[k]; target = nb_part[k]; }
    return target < 0 ? 0 : best - own;
  };
  std::vector<char> locked(nc, 0);
  for (int pass = 0; pass < 8; ++pass) {
    // max-heap of (gain, -cell) with lazy invalidation by a per-cell stamp
    std::vector<std::tuple<int, int64_t, int64_t>> heap;  // gain, -cell, stamp
    std::vector<int64_t> stamp(nc, 0);
    auto push = [&](int64_t i) {
      int t;
      const int g = best_move(i, t);
      if (t >= 0) {
        heap.emplace_back(g, -i, ++stamp[i]);
        std::push_heap(heap.begin(), heap.end());
      }
    };
    for (int64_t i = 0; i < nc; ++i) push(i);
    std::fill(locked.begin(), locked.end(), 0);
    std::vector<std::pair<int64_t, int>> moves;  // (cell, previous part)
    int64_t cum = 0, best_cum = 0;
    size_t best_len = 0;
    const size_t max_moves = heap.size();
    while (!heap.empty() && moves.size() < max_moves) {
      std::pop_heap(heap.begin(), heap.end());
      auto [g, mi, st] = heap.back();
      heap.pop_back();
      const int64_t i = -mi;
      if (locked[i] || st != stamp[i]) continue;
      int t;
      const int g2 = best_move(i, t);
      if (t < 0 || g2 != g) continue;
      const int p = gm.part[i];
      if (size[t] + 1 > hi || size[p] - 1 < lo) continue;
      gm.part[i] = t;
      --size[p];
      ++size[t];
      locked[i] = 1;
      moves.emplace_back(i, p);
      cum += g;
      if (cum > best_cum) { best_cum = cum; best_len = moves.size(); }
      for (int q = 0; q < nfc; ++q) {
        const int64_t j = gm.nbr_id[i * 6 + q];
        if (j >= 0 && j < nc && !locked[j]) push(j);
      }
      if (cum < best_cum - 64) break;  // a long losing streak: stop the pass early
    }
    for (size_t k = moves.size(); k > best_len; --k) {  // roll back to the best prefix
      const auto [i, p] = moves[k - 1];
      --size[gm.part[i]];
      ++size[p];
      gm.part[i] = p;
    }
    if (best_cum <= 0) break;
  }
}

// ============================================================================
// Geometry, faces, periodic pairing, boundary ghosts, neighbours and Alg. 1 stencils of a
// mesh (the whole mesh, or one rank's region of it).  open_ok[i]: cell i may keep faces
// without a partner (the outer rim of a region; such faces are left out); stencil_ok[i]:
// build cell i's stencils (cells without them are never reconstructed).  NULL = every cell.
static void build_core(GlobalMesh& gm, const double* xyz, int64_t n_nodes, const int8_t* type, const int64_t* cn,
                       int64_t n_cells, const double* per_origin, const double* per_len,
                       const int64_t* bface_nodes, const int32_t* bface_tag, int64_t n_bf,
                       const std::vector<char>* open_ok, const std::vector<char>* stencil_ok,
                       bool hybrid = false) {
  PhaseTimer pt("mesh core");
  if (n_cells <= 0 || n_nodes <= 0 || !xyz || !type || !cn) throw Error(1, "empty mesh");
  gm.nc = n_cells;
  gm.type.assign(type, type + n_cells);
  // single-kind tet or hex meshes, or hybrid tet/prism meshes (f4, R30; hybrid: the whole
  // mesh has prisms, so a region without any gets the same layout as the others)
  bool any_prism = hybrid;
  for (int64_t i = 0; i < n_cells; ++i) any_prism |= type[i] == 6;
  const int ct = any_prism ? 6 : type[0];
  Layout& L = gm.lay;
  L.cell_type = ct;
  L.nfaces = cell_nfaces(ct);
  L.ngp = ct == 4 ? 3 : 4;
  L.nv = ct == 4 ? 3 : 4;
  // sub-stencils: tets 4 (R16, up to 6 members; 7 next to a prism), prisms 6 (R30), hexes 8
  L.M = ct == 4 ? 4 : (ct == 6 ? 6 : 8);
  L.NM = ct == 4 ? 6 : (ct == 6 ? 7 : 3);
  for (int a = 0; a < 3; ++a) gm.per_len[a] = per_len ? per_len[a] : 0.0;
  const double O[3] = {per_origin ? per_origin[0] : 0.0, per_origin ? per_origin[1] : 0.0,
                       per_origin ? per_origin[2] : 0.0};
  auto node = [&](int64_t id) { return P3{xyz[3 * id], xyz[3 * id + 1], xyz[3 * id + 2]}; };
  const int nfc = L.nfaces;  // half-face stride per cell (cells of a hybrid mesh use their first nf(i))
  auto nf_of = [&](int64_t i) { return cell_nfaces(type[i]); };
  // node ids of face p of cell i, returns its vertex count
  auto fnodes = [&](int64_t i, int p, int64_t nd[4]) {
    int sl[4];
    const int nv = face_slots(type[i], p, sl);
    for (int q = 0; q < nv; ++q) nd[q] = cn[i * 8 + sl[q]];
    return nv;
  };
  // ---------------- geometry ----------------
  gm.V.resize(n_cells);
  gm.C.resize(3 * n_cells);
  gm.M2.resize(6 * n_cells);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_cells; ++i) {
    P3 v[8];
    for (int k = 0; k < type[i]; ++k) v[k] = node(cn[i * 8 + k]);
    double V;
    P3 c;
    cell_geometry(type[i], v, V, c, &gm.M2[6 * i]);
    gm.V[i] = V;
    gm.C[3 * i] = c.x; gm.C[3 * i + 1] = c.y; gm.C[3 * i + 2] = c.z;
  }
  for (int64_t i = 0; i < n_cells; ++i)
    if (!(gm.V[i] > 0)) throw Error(2, "degenerate cell " + std::to_string(i));
  auto centroid = [&](int64_t i) { return P3{gm.C[3 * i], gm.C[3 * i + 1], gm.C[3 * i + 2]}; };

  pt.lap("geometry");
  // ---------------- faces: bucket half-faces by their smallest node ----------
  // half-face h = i * nfc + p; p >= nf(i) (a tet in a hybrid mesh) is no face (key -1)
  const int64_t nh = n_cells * nfc;
  std::vector<std::array<int64_t, 4>> hkey(nh);
  int64_t nh_valid = 0;
  for (int64_t i = 0; i < n_cells; ++i)
    for (int p = 0; p < nfc; ++p) {
      std::array<int64_t, 4> k{INT64_MAX, INT64_MAX, INT64_MAX, INT64_MAX};
      if (p < nf_of(i)) {
        int64_t nd[4];
        const int nv = fnodes(i, p, nd);
        for (int q = 0; q < nv; ++q) k[q] = nd[q];
        std::sort(k.begin(), k.end());
        ++nh_valid;
      } else {
        k[0] = -1;
      }
      hkey[i * nfc + p] = k;
    }
  std::vector<int64_t> bstart(n_nodes + 1, 0), order(nh_valid);
  for (int64_t h = 0; h < nh; ++h)
    if (hkey[h][0] >= 0) bstart[hkey[h][0] + 1]++;
  for (int64_t n = 0; n < n_nodes; ++n) bstart[n + 1] += bstart[n];
  {
    std::vector<int64_t> fill(bstart.begin(), bstart.end() - 1);
    for (int64_t h = 0; h < nh; ++h)
      if (hkey[h][0] >= 0) order[fill[hkey[h][0]]++] = h;  // stable: ascending h
  }
  // boundary tags by key
  std::unordered_map<std::string, int32_t> btag;
  auto key_str = [](const std::array<int64_t, 4>& k) { return std::string((const char*)k.data(), sizeof(int64_t) * 4); };
  for (int64_t b = 0; b < n_bf; ++b) {
    std::array<int64_t, 4> k{INT64_MAX, INT64_MAX, INT64_MAX, INT64_MAX};
    int q = 0;
    for (int j = 0; j < 4; ++j)
      if (bface_nodes[b * 4 + j] >= 0) k[q++] = bface_nodes[b * 4 + j];
    std::sort(k.begin(), k.end());
    btag[key_str(k)] = bface_tag[b];
  }
  gm.cell_face.assign(n_cells * 6, -1);
  std::vector<int64_t> unmatched;
  struct FaceTmp {
    int64_t owner, nb, hown;
    int32_t bc;
    P3 shift;
  };
  std::vector<FaceTmp> ft;
  ft.reserve(nh / 2 + 16);
  for (int64_t n = 0; n < n_nodes; ++n) {
    int64_t b0 = bstart[n], b1 = bstart[n + 1];
    std::sort(order.begin() + b0, order.begin() + b1, [&](int64_t a, int64_t b) {
      return hkey[a] != hkey[b] ? hkey[a] < hkey[b] : a < b;
    });
    for (int64_t j = b0; j < b1;) {
      int64_t e = j + 1;
      while (e < b1 && hkey[order[e]] == hkey[order[j]]) ++e;
      if (e - j > 2) throw Error(2, "non-manifold face at cell " + std::to_string(order[j] / nfc));
      if (e - j == 2) {
        int64_t ha = order[j], hb = order[j + 1];  // ha < hb => lower cell id is the owner (R19)
        ft.push_back({ha / nfc, hb / nfc, ha, 0, {0, 0, 0}});
        gm.cell_face[(ha / nfc) * 6 + ha % nfc] = (int64_t)ft.size() - 1;
        gm.cell_face[(hb / nfc) * 6 + hb % nfc] = (int64_t)ft.size() - 1;
      } else {
        int64_t ha = order[j];
        auto it = btag.find(key_str(hkey[ha]));
        if (it != btag.end()) {
          ft.push_back({ha / nfc, -1, ha, it->second, {0, 0, 0}});
          gm.cell_face[(ha / nfc) * 6 + ha % nfc] = (int64_t)ft.size() - 1;
        } else {
          unmatched.push_back(ha);
        }
      }
      j = e;
    }
  }
  // periodic pairing (R23): canonical wrapped vertex coordinates
  if (!unmatched.empty()) {
    // (region rims of a non-periodic mesh: handled by the check below)
    double Lm = std::max(gm.per_len[0], std::max(gm.per_len[1], gm.per_len[2]));
    if (!(Lm > 0)) {
      for (int64_t h : unmatched)
        if (!open_ok || !(*open_ok)[h / nfc]) throw Error(2, "open boundary face at cell " + std::to_string(h / nfc));
      unmatched.clear();
    }
    const double tol = 1e-7 * Lm;
    struct PK {
      std::array<int64_t, 12> k;
      int64_t h;
    };
    std::vector<PK> pk(unmatched.size());
    for (size_t u = 0; u < unmatched.size(); ++u) {
      int64_t h = unmatched[u];
      std::array<std::array<int64_t, 3>, 4> q;
      for (int a = 0; a < 4; ++a) q[a] = {INT64_MAX, INT64_MAX, INT64_MAX};
      int64_t fn[4];
      const int nvh = fnodes(h / nfc, (int)(h % nfc), fn);
      for (int v = 0; v < nvh; ++v) {
        int64_t nd = fn[v];
        double c3[3] = {xyz[3 * nd] - O[0], xyz[3 * nd + 1] - O[1], xyz[3 * nd + 2] - O[2]};
        for (int a = 0; a < 3; ++a) {
          double y = c3[a];
          if (gm.per_len[a] > 0) {
            y -= gm.per_len[a] * std::floor(y / gm.per_len[a]);
            if (gm.per_len[a] - y < tol) y = 0.0;
          }
          q[v][a] = (int64_t)std::llround(y / tol);
        }
      }
      std::sort(q.begin(), q.end());
      for (int v = 0; v < 4; ++v)
        for (int a = 0; a < 3; ++a) pk[u].k[v * 3 + a] = q[v][a];
      pk[u].h = h;
    }
    std::sort(pk.begin(), pk.end(), [](const PK& a, const PK& b) { return a.k != b.k ? a.k < b.k : a.h < b.h; });
    for (size_t u = 0; u < pk.size(); u += 2) {
      if (u + 1 >= pk.size() || pk[u].k != pk[u + 1].k || (u + 2 < pk.size() && pk[u + 2].k == pk[u].k)) {
        // a region's rim: the partner lies outside the region (left open)
        if (open_ok && (*open_ok)[pk[u].h / nfc] && (u + 1 >= pk.size() || pk[u].k != pk[u + 1].k)) {
          --u;
          continue;
        }
        throw Error(2, "unmatched boundary face at cell " + std::to_string(pk[u].h / nfc));
      }
      int64_t ha = pk[u].h, hb = pk[u + 1].h;
      if (hb / nfc < ha / nfc) std::swap(ha, hb);
      if (ha / nfc == hb / nfc) throw Error(2, "self-periodic cell " + std::to_string(ha / nfc));
      // shift = (owner face centroid) - (neighbour face centroid), snapped to the box lengths
      P3 ca{0, 0, 0}, cb{0, 0, 0};
      int64_t fa[4], fb[4];
      const int nva = fnodes(ha / nfc, (int)(ha % nfc), fa);
      fnodes(hb / nfc, (int)(hb % nfc), fb);
      for (int v = 0; v < nva; ++v) {
        ca = ca + (1.0 / nva) * node(fa[v]);
        cb = cb + (1.0 / nva) * node(fb[v]);
      }
      P3 d = ca - cb;
      double s[3] = {d.x, d.y, d.z};
      for (int a = 0; a < 3; ++a) s[a] = gm.per_len[a] > 0 ? gm.per_len[a] * std::round(s[a] / gm.per_len[a]) : 0.0;
      ft.push_back({ha / nfc, hb / nfc, ha, 0, {s[0], s[1], s[2]}});
      gm.cell_face[(ha / nfc) * 6 + ha % nfc] = (int64_t)ft.size() - 1;
      gm.cell_face[(hb / nfc) * 6 + hb % nfc] = (int64_t)ft.size() - 1;
    }
  }
  // canonical face order: by (owner, owner-local face index)
  {
    std::vector<int64_t> perm(ft.size());
    std::iota(perm.begin(), perm.end(), 0);
    std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return ft[a].hown < ft[b].hown; });
    std::vector<int64_t> inv(ft.size());
    for (size_t k = 0; k < perm.size(); ++k) inv[perm[k]] = (int64_t)k;
    std::vector<FaceTmp> f2(ft.size());
    for (size_t k = 0; k < perm.size(); ++k) f2[k] = ft[perm[k]];
    ft.swap(f2);
    for (auto& f : gm.cell_face)
      if (f >= 0) f = inv[f];
  }
  gm.nf = (int64_t)ft.size();
  gm.f_owner.resize(gm.nf);
  gm.f_nb.resize(gm.nf);
  gm.f_bc.resize(gm.nf);
  gm.f_ghost.assign(gm.nf, -1);
  gm.f_shift.resize(3 * gm.nf);
  gm.f_vert.assign(12 * gm.nf, 0.0);
  gm.f_nv.resize(gm.nf);
  gm.f_area.resize(gm.nf);
  for (int64_t f = 0; f < gm.nf; ++f) {
    const FaceTmp& F = ft[f];
    gm.f_owner[f] = F.owner;
    gm.f_nb[f] = F.nb;
    gm.f_bc[f] = F.bc;
    gm.f_shift[3 * f] = F.shift.x; gm.f_shift[3 * f + 1] = F.shift.y; gm.f_shift[3 * f + 2] = F.shift.z;
    int p = (int)(F.hown % nfc);
    P3 v[4];
    int64_t fn[4];
    const int nvf = fnodes(F.owner, p, fn);
    gm.f_nv[f] = (int8_t)nvf;
    for (int q = 0; q < nvf; ++q) v[q] = node(fn[q]);
    // orient out of the owner
    P3 fc{0, 0, 0};
    for (int q = 0; q < nvf; ++q) fc = fc + (1.0 / nvf) * v[q];
    P3 nn = nvf == 3 ? crossp(v[1] - v[0], v[2] - v[0]) : crossp(v[2] - v[0], v[3] - v[1]);
    if (dotp(nn, fc - centroid(F.owner)) < 0) {
      if (nvf == 3) std::swap(v[1], v[2]);
      else std::swap(v[1], v[3]);
    }
    for (int q = 0; q < nvf; ++q) {
      gm.f_vert[12 * f + 3 * q] = v[q].x; gm.f_vert[12 * f + 3 * q + 1] = v[q].y; gm.f_vert[12 * f + 3 * q + 2] = v[q].z;
    }
    P3 gx[4], gn[4];
    double gw[4];
    int ng = face_gps(nvf, v, gx, gn, gw);
    double a = 0;
    for (int g = 0; g < ng; ++g) a += gw[g];
    gm.f_area[f] = a;
  }
  for (int64_t i = 0; i < n_cells; ++i)
    for (int p = 0; p < nf_of(i); ++p)
      if (gm.cell_face[i * 6 + p] < 0 && !(open_ok && (*open_ok)[i]))
        throw Error(2, "open face at cell " + std::to_string(i));
  pt.lap("faces + periodic pairing");
  // ---------------- boundary ghosts (R25) ----------------
  for (int64_t f = 0; f < gm.nf; ++f) {
    if (gm.f_nb[f] >= 0) continue;
    int64_t g = gm.ng++;
    gm.f_ghost[f] = (int32_t)g;
    gm.g_cell.push_back(gm.f_owner[f]);
    gm.g_face.push_back(f);
    gm.g_bc.push_back(gm.f_bc[f]);
    P3 v[4];
    const int nvf = gm.f_nv[f];
    for (int q = 0; q < nvf; ++q) v[q] = {gm.f_vert[12 * f + 3 * q], gm.f_vert[12 * f + 3 * q + 1], gm.f_vert[12 * f + 3 * q + 2]};
    P3 gx[4], gn[4];
    double gw[4];
    int ngp = face_gps(nvf, v, gx, gn, gw);
    P3 xf{0, 0, 0}, nf{0, 0, 0};
    for (int q = 0; q < ngp; ++q) {
      xf = xf + (gw[q] / gm.f_area[f]) * gx[q];
      nf = nf + gw[q] * gn[q];
    }
    nf = (1.0 / len(nf)) * nf;
    P3 ci = centroid(gm.f_owner[f]);
    P3 cg = ci - (2.0 * dotp(ci - xf, nf)) * nf;
    gm.gV.push_back(gm.V[gm.f_owner[f]]);
    gm.gC.push_back(cg.x); gm.gC.push_back(cg.y); gm.gC.push_back(cg.z);
    gm.g_normal.push_back(nf.x); gm.g_normal.push_back(nf.y); gm.g_normal.push_back(nf.z);
    // reflected second moments R M2 R, R = I - 2 n n^T
    const double* m = &gm.M2[6 * gm.f_owner[f]];
    double S[3][3] = {{m[0], m[3], m[4]}, {m[3], m[1], m[5]}, {m[4], m[5], m[2]}};
    double n3[3] = {nf.x, nf.y, nf.z}, R[3][3], T[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) R[a][b] = (a == b) - 2.0 * n3[a] * n3[b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) s += R[a][k] * S[k][l] * R[b][l];
        T[a][b] = s;
      }
    gm.gM2.push_back(T[0][0]); gm.gM2.push_back(T[1][1]); gm.gM2.push_back(T[2][2]);
    gm.gM2.push_back(T[0][1]); gm.gM2.push_back(T[0][2]); gm.gM2.push_back(T[1][2]);
  }
  pt.lap("boundary ghosts");
  // ---------------- CellNeighbor and h for dt ----------------
  gm.nbr_id.assign(n_cells * 6, -1);
  gm.nbr_shift.assign(n_cells * 18, 0.0);
  gm.h_dt.resize(n_cells);
  for (int64_t i = 0; i < n_cells; ++i) {
    double smax = 0;
    for (int p = 0; p < nf_of(i); ++p) {
      int64_t f = gm.cell_face[i * 6 + p];
      if (f < 0) continue;  // region rim (open_ok): no neighbour, never used
      smax = std::max(smax, gm.f_area[f]);
      double sg = 1.0;
      int64_t other;
      if (gm.f_nb[f] < 0) {
        other = n_cells + gm.f_ghost[f];
        sg = 0.0;
      } else if (gm.f_owner[f] == i) {
        other = gm.f_nb[f];
      } else {
        other = gm.f_owner[f];
        sg = -1.0;
      }
      gm.nbr_id[i * 6 + p] = other;
      for (int a = 0; a < 3; ++a) gm.nbr_shift[i * 18 + p * 3 + a] = sg * gm.f_shift[3 * f + a];
    }
    gm.h_dt[i] = smax > 0 ? gm.V[i] / smax : 0.0;
  }
  pt.lap("neighbours, h");
  // ---------------- Alg. 1 stencils + sub-stencils ----------------
  gm.big_off.assign(n_cells + 1, 0);
  std::vector<std::vector<Member>> big(n_cells);
  gm.sub_slot.assign(n_cells * L.M * L.NM, (int8_t)-1);
  int max_k = 0;
  bool bad = false;
  int64_t bad_cell = -1;
  int bad_code = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(max : max_k)
  for (int64_t i = 0; i < n_cells; ++i) {
    if (stencil_ok && !(*stencil_ok)[i]) continue;
    std::vector<Member>& S = big[i];
    int err = 0;
    auto add = [&](int64_t id, P3 s) {
      if (id == i) {
        if (!same_shift(s, {0, 0, 0})) err = 1;
        return;
      }
      for (auto& m : S)
        if (m.id == id) {
          if (!same_shift(m.s, s)) err = 1;
          return;
        }
      S.push_back({id, s});
    };
    auto nb = [&](int64_t c, int p) {
      return Member{gm.nbr_id[c * 6 + p], {gm.nbr_shift[c * 18 + 3 * p], gm.nbr_shift[c * 18 + 3 * p + 1], gm.nbr_shift[c * 18 + 3 * p + 2]}};
    };
    for (int p = 0; p < nf_of(i); ++p) {
      Member m = nb(i, p);
      add(m.id, m.s);
    }
    for (int p = 0; p < nf_of(i); ++p) {
      Member m = nb(i, p);
      if (m.id >= n_cells) continue;  // ghosts have no neighbours
      for (int q = 0; q < nf_of(m.id); ++q) {
        Member m2 = nb(m.id, q);
        add(m2.id, m.s + m2.s);
      }
    }
    if ((int)S.size() > kMaxStencil) err = 2;
    auto slot_of = [&](int64_t id) -> int {
      for (size_t k = 0; k < S.size(); ++k)
        if (S[k].id == id) return (int)k;
      return -1;
    };
    int8_t* ss = &gm.sub_slot[i * L.M * L.NM];
    if (type[i] == 4) {
      // R16: sub m = three face neighbours {T_m} + neighbours of i_m
      const int tri[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {2, 0, 3}};
      for (int m = 0; m < 4; ++m) {
        int cnt = 0;
        auto put = [&](int64_t id) {
          if (id == i) return;
          int s = slot_of(id);
          for (int k = 0; k < cnt; ++k)
            if (ss[m * L.NM + k] == s) return;
          if (cnt < L.NM) ss[m * L.NM + cnt++] = (int8_t)s;
          else err = 3;
        };
        for (int k = 0; k < 3; ++k) put(gm.nbr_id[i * 6 + tri[m][k]]);
        int64_t im = gm.nbr_id[i * 6 + m];
        if (im < n_cells)
          for (int q = 0; q < nf_of(im); ++q) put(gm.nbr_id[im * 6 + q]);
      }
    } else if (type[i] == 6) {
      // R30: the triangle-face neighbour (face 0 or 1) and two ring-adjacent side neighbours
      const int ps[6][3] = {{0, 2, 3}, {0, 3, 4}, {0, 4, 2}, {1, 2, 3}, {1, 3, 4}, {1, 4, 2}};
      for (int m = 0; m < 6; ++m)
        for (int k = 0; k < 3; ++k) ss[m * L.NM + k] = (int8_t)slot_of(gm.nbr_id[i * 6 + ps[m][k]]);
    } else {
      const int hs[8][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 4}, {0, 4, 1}, {5, 1, 2}, {5, 2, 3}, {5, 3, 4}, {5, 4, 1}};
      for (int m = 0; m < 8; ++m)
        for (int k = 0; k < 3; ++k) ss[m * 3 + k] = (int8_t)slot_of(gm.nbr_id[i * 6 + hs[m][k]]);
    }
    if (err) {
#pragma omp critical
      {
        bad = true;
        if (bad_cell < 0 || i < bad_cell) {
          bad_cell = i;
          bad_code = err;
        }
      }
    }
    max_k = std::max(max_k, (int)S.size());
  }
  if (bad)
    throw Error(2, bad_code == 1 ? "periodic box too small for the two-layer stencil at cell " + std::to_string(bad_cell)
                                 : "stencil capacity exceeded at cell " + std::to_string(bad_cell));
  for (int64_t i = 0; i < n_cells; ++i) gm.big_off[i + 1] = gm.big_off[i] + (int64_t)big[i].size();
  gm.big_id.resize(gm.big_off[n_cells]);
  gm.big_shift.resize(3 * gm.big_off[n_cells]);
  for (int64_t i = 0; i < n_cells; ++i)
    for (size_t k = 0; k < big[i].size(); ++k) {
      int64_t o = gm.big_off[i] + (int64_t)k;
      gm.big_id[o] = big[i][k].id;
      gm.big_shift[3 * o] = big[i][k].s.x; gm.big_shift[3 * o + 1] = big[i][k].s.y; gm.big_shift[3 * o + 2] = big[i][k].s.z;
    }
  {
    // pad the stencil width to a capacity the reconstruction kernel is compiled for
    // (hybrid meshes: 20 and up)
    const int caps[] = {14, 16, 20, 24, 32, 40};
    L.K = 40;
    for (int c : caps)
      if (c >= max_k && (ct != 6 || c >= 20)) {
        L.K = c;
        break;
      }
  }
  pt.lap("stencils");
}

// recursive coordinate bisection on centroids C [n][3] (P:730-739 objective: balance,
// small interfaces); splits proportional to the rank counts on each side
static void rcb_partition(const double* C, int64_t n, int nr, int32_t* part) {
  std::vector<int64_t> ids(n);
  std::iota(ids.begin(), ids.end(), 0);
  struct Task {
    int64_t b, e;
    int r0, nr;
  };
  std::vector<Task> st{{0, n, 0, nr}};
  while (!st.empty()) {
    Task t = st.back();
    st.pop_back();
    if (t.nr == 1) {
      for (int64_t k = t.b; k < t.e; ++k) part[ids[k]] = t.r0;
      continue;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t k = t.b; k < t.e; ++k)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], C[3 * ids[k] + a]);
        hi[a] = std::max(hi[a], C[3 * ids[k] + a]);
      }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
      if (hi[a] - lo[a] > hi[ax] - lo[ax] + 1e-12) ax = a;
    int nl = t.nr / 2;
    int64_t cut = t.b + (t.e - t.b) * nl / t.nr;
    std::nth_element(ids.begin() + t.b, ids.begin() + cut, ids.begin() + t.e, [&](int64_t a, int64_t b) {
      double xa = C[3 * a + ax], xb = C[3 * b + ax];
      return xa != xb ? xa < xb : a < b;
    });
    st.push_back({t.b, cut, t.r0, nl});
    st.push_back({cut, t.e, t.r0 + nl, t.nr - nl});
  }
}

// accepted: tet-only, hex-only, or tets and prisms mixed (hybrid, f4)
static void check_cells(const int8_t* type, const int64_t* cn, int64_t n_cells, int64_t n_nodes) {
  const bool hex = type[0] == 8;
  for (int64_t i = 0; i < n_cells; ++i) {
    const int t = type[i];
    if (t != 4 && t != 6 && t != 8) throw Error(2, "unsupported element at cell " + std::to_string(i));
    if ((t == 8) != hex)
      throw Error(2, "hexes cannot be mixed with other element kinds (cell " + std::to_string(i) + ")");
    for (int k = 0; k < t; ++k) {
      int64_t v = cn[i * 8 + k];
      if (v < 0 || v >= n_nodes) throw Error(2, "invalid node id in cell " + std::to_string(i));
    }
  }
}

static void centroid_bbox(GlobalMesh& gm, const double* C, int64_t n) {
  for (int a = 0; a < 3; ++a) {
    gm.bbox_lo[a] = 1e300;
    gm.bbox_hi[a] = -1e300;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      gm.bbox_lo[a] = std::min(gm.bbox_lo[a], C[3 * i + a]);
      gm.bbox_hi[a] = std::max(gm.bbox_hi[a], C[3 * i + a]);
    }
}

// One rank's region of a partitioned mesh (rank_only > 0): the rank's owned cells and every
// cell within four node-adjacency layers of them (a superset of the 3 face-adjacency ghost
// layers, and of their face partners), found by streaming passes over the cell
// list with a bitmap of (periodically identified) nodes.  Host memory is O(region): the
// only per-global-cell arrays are the centroids and the partition (28 bytes per cell).
static GlobalMesh build_region(const double* xyz, int64_t n_nodes, const int8_t* type, const int64_t* cn,
                               int64_t n_cells, const double* per_origin, const double* per_len,
                               const int64_t* bface_nodes, const int32_t* bface_tag, int64_t n_bf, int32_t n_ranks,
                               const int32_t* cell_part, int rank) {
  PhaseTimer pt("region");
  // centroids of every cell (the partition input), the same numbers as the whole-mesh build
  std::vector<double> C(3 * n_cells);
  std::vector<int32_t> part(n_cells, 0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_cells; ++i) {
    P3 v[8];
    for (int k = 0; k < type[i]; ++k) v[k] = {xyz[3 * cn[i * 8 + k]], xyz[3 * cn[i * 8 + k] + 1], xyz[3 * cn[i * 8 + k] + 2]};
    double V, m2[6];
    P3 c;
    cell_geometry(type[i], v, V, c, m2);
    C[3 * i] = c.x; C[3 * i + 1] = c.y; C[3 * i + 2] = c.z;
  }
  GlobalMesh gm;
  centroid_bbox(gm, C.data(), n_cells);
  if (cell_part) {
    for (int64_t i = 0; i < n_cells; ++i) {
      if (cell_part[i] < 0 || cell_part[i] >= n_ranks) throw Error(1, "cell_part out of range at cell " + std::to_string(i));
      part[i] = cell_part[i];
    }
  } else {
    rcb_partition(C.data(), n_cells, n_ranks, part.data());
  }
  pt.lap("centroids + partition");
  // periodically identified node ids: wrapped coordinates quantised (R23)
  std::vector<int64_t> canon(n_nodes);
  {
    double Lm = std::max(per_len ? per_len[0] : 0.0, std::max(per_len ? per_len[1] : 0.0, per_len ? per_len[2] : 0.0));
    if (!(Lm > 0)) {
      std::iota(canon.begin(), canon.end(), 0);
    } else {
      const double tol = 1e-7 * Lm;
      std::vector<std::pair<std::array<int64_t, 3>, int64_t>> key(n_nodes);
#pragma omp parallel for schedule(static)
      for (int64_t nd = 0; nd < n_nodes; ++nd) {
        std::array<int64_t, 3> q;
        for (int a = 0; a < 3; ++a) {
          double y = xyz[3 * nd + a] - (per_origin ? per_origin[a] : 0.0);
          if (per_len[a] > 0) {
            y -= per_len[a] * std::floor(y / per_len[a]);
            if (per_len[a] - y < tol) y = 0.0;
          }
          q[a] = (int64_t)std::llround(y / tol);
        }
        key[nd] = {q, nd};
      }
      std::sort(key.begin(), key.end());
      int64_t id = -1;
      for (int64_t k = 0; k < n_nodes; ++k) {
        if (k == 0 || key[k].first != key[k - 1].first) id = key[k].second;
        canon[key[k].second] = id;
      }
    }
  }
  // region: owned cells, then four node-adjacency layers
  std::vector<int8_t> lay(n_cells, -1);
  for (int64_t i = 0; i < n_cells; ++i)
    if (part[i] == rank) lay[i] = 0;
  std::vector<char> mark(n_nodes, 0);
  for (int l = 1; l <= 4; ++l) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_cells; ++i)
      if (lay[i] == l - 1)
        for (int k = 0; k < type[i]; ++k) mark[canon[cn[i * 8 + k]]] = 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_cells; ++i) {
      if (lay[i] >= 0) continue;
      for (int k = 0; k < type[i]; ++k)
        if (mark[canon[cn[i * 8 + k]]]) {
          lay[i] = (int8_t)l;
          break;
        }
    }
  }
  std::vector<int64_t> R;
  for (int64_t i = 0; i < n_cells; ++i)
    if (lay[i] >= 0) R.push_back(i);
  if (R.empty() || std::none_of(R.begin(), R.end(), [&](int64_t i) { return lay[i] == 0; }))
    throw Error(1, "rank " + std::to_string(rank) + " owns no cells");
  pt.lap("region (4 node layers)");
  const int64_t nr = (int64_t)R.size();
  std::vector<int64_t> sub_cn((size_t)nr * 8);
  std::vector<int8_t> sub_type(nr);
  std::vector<char> open_ok(nr), stencil_ok(nr);
  for (int64_t k = 0; k < nr; ++k) {
    std::memcpy(&sub_cn[8 * k], cn + 8 * R[k], 8 * sizeof(int64_t));
    sub_type[k] = type[R[k]];
    open_ok[k] = lay[R[k]] == 4;       // every face of layers <= 3 has its partner in the region
    stencil_ok[k] = lay[R[k]] <= 1;    // owned + face layer 1 (reconstructed cells)
  }
  const bool hybrid = std::any_of(type, type + n_cells, [](int8_t t) { return t == 6; });
  build_core(gm, xyz, n_nodes, sub_type.data(), sub_cn.data(), nr, per_origin, per_len, bface_nodes, bface_tag,
             n_bf, &open_ok, &stencil_ok, hybrid);
  gm.gid = R;
  gm.nc_global = n_cells;
  gm.n_ranks = n_ranks;
  gm.only_rank = rank;
  gm.part.resize(nr);
  for (int64_t k = 0; k < nr; ++k) gm.part[k] = part[R[k]];
  gm.edge_cut = -1;  // global cut unknown in a region build; rank_cut_faces in the plan
  pt.lap("region mesh");
  return gm;
}

GlobalMesh build_global_mesh(const double* xyz, int64_t n_nodes, const int8_t* type, const int64_t* cn,
                             int64_t n_cells, const double* per_origin, const double* per_len,
                             const int64_t* bface_nodes, const int32_t* bface_tag, int64_t n_bf, int32_t n_ranks,
                             const int32_t* cell_part, int32_t rank_only) {
  if (n_cells <= 0 || n_nodes <= 0 || !xyz || !type || !cn) throw Error(1, "empty mesh");
  check_cells(type, cn, n_cells, n_nodes);
  if (n_ranks > 1 && rank_only > 0) {
    if (rank_only > n_ranks) throw Error(1, "rank_only out of range");
    return build_region(xyz, n_nodes, type, cn, n_cells, per_origin, per_len, bface_nodes, bface_tag, n_bf, n_ranks,
                        cell_part, rank_only - 1);
  }
  GlobalMesh gm;
  PhaseTimer pt("global mesh");
  build_core(gm, xyz, n_nodes, type, cn, n_cells, per_origin, per_len, bface_nodes, bface_tag, n_bf, nullptr, nullptr);
  gm.nc_global = n_cells;
  centroid_bbox(gm, gm.C.data(), n_cells);
  const int nfc = gm.lay.nfaces;
  // ---------------- partition (a3) ----------------
  gm.n_ranks = std::max(1, n_ranks);
  gm.part.assign(n_cells, 0);
  if (gm.n_ranks > 1) {
    if (cell_part) {
      for (int64_t i = 0; i < n_cells; ++i) {
        if (cell_part[i] < 0 || cell_part[i] >= gm.n_ranks) throw Error(1, "cell_part out of range at cell " + std::to_string(i));
        gm.part[i] = cell_part[i];
      }
    } else {
      rcb_partition(gm.C.data(), n_cells, gm.n_ranks, gm.part.data());
      auto cut = [&] {
        int64_t c = 0;
        for (int64_t f = 0; f < gm.nf; ++f)
          if (gm.f_nb[f] >= 0 && gm.part[gm.f_owner[f]] != gm.part[gm.f_nb[f]]) ++c;
        return c;
      };
      gm.edge_cut_rcb = cut();
      refine_partition(gm, nfc);
    }
    for (int64_t f = 0; f < gm.nf; ++f)
      if (gm.f_nb[f] >= 0 && gm.part[gm.f_owner[f]] != gm.part[gm.f_nb[f]]) ++gm.edge_cut;
  }
  pt.lap("partition");
  return gm;
}

// ============================================================================
// Per-rank plan: owned cells (Morton order), 3 ghost layers grouped by owner
// rank, device arrays in entry-major layout.
// Least-squares operators of cell i (a2, P:432-442 with the scaled basis of R20),
// written to op[E] in the global-table order: A0+ (9 x K, row d, /h^|d|) then the
// sub-stencil pseudo-inverses (M x 3 x NM, /h).  Entries of absent members stay 0.
// Returns false for a rank-deficient system.
static bool cell_operators(const GlobalMesh& gm, int64_t i, double* op) {
  const Layout& L = gm.lay;
  const int64_t n_cells = gm.nc;
  const int E = L.op_entries();
  for (int e = 0; e < E; ++e) op[e] = 0.0;
  const int64_t o0 = gm.big_off[i];
  const int K = (int)(gm.big_off[i + 1] - o0);
  if (K > 64 || K < 9) return false;
  const double h = std::cbrt(gm.V[i]);
  const P3 ci{gm.C[3 * i], gm.C[3 * i + 1], gm.C[3 * i + 2]};
  const double* mi = &gm.M2[6 * i];
  // rows: member image centroid offset D and zero-mean quadratic moments (A.4)
  double A[64 * 9];
  for (int k = 0; k < K; ++k) {
    int64_t id = gm.big_id[o0 + k];
    P3 ck;
    const double* mk;
    if (id < n_cells) {
      ck = {gm.C[3 * id], gm.C[3 * id + 1], gm.C[3 * id + 2]};
      mk = &gm.M2[6 * id];
    } else {
      int64_t g = id - n_cells;
      ck = {gm.gC[3 * g], gm.gC[3 * g + 1], gm.gC[3 * g + 2]};
      mk = &gm.gM2[6 * g];
    }
    P3 D = (ck + P3{gm.big_shift[3 * (o0 + k)], gm.big_shift[3 * (o0 + k) + 1], gm.big_shift[3 * (o0 + k) + 2]}) - ci;
    double* r = &A[k * 9];
    r[0] = D.x / h; r[1] = D.y / h; r[2] = D.z / h;
    const double h2 = h * h;
    r[3] = (mk[0] + D.x * D.x - mi[0]) / h2;
    r[4] = (mk[1] + D.y * D.y - mi[1]) / h2;
    r[5] = (mk[2] + D.z * D.z - mi[2]) / h2;
    r[6] = (mk[3] + D.x * D.y - mi[3]) / h2;
    r[7] = (mk[4] + D.x * D.z - mi[4]) / h2;
    r[8] = (mk[5] + D.y * D.z - mi[5]) / h2;
  }
  double P[9 * 64];
  if (!pinv_qr(K, 9, A, P)) return false;
#if HGKS_RECON_NE
  {
    // normal equations of the scaled system: G = A^T A = L L^T, W = L^{-1} (lower), so the
    // scaled coefficients are W^T W A^T dq; the device rebuilds the rows of A from member
    // geometry and stores only W.  Checked against the QR pseudo-inverse (cond(G) =
    // cond(A)^2 is ~1e2-2e3 on these stencils).
    double G[9][9] = {}, Lc[9][9] = {}, Wm[9][9] = {};
    for (int a = 0; a < 9; ++a)
      for (int b = 0; b < 9; ++b)
        for (int k = 0; k < K; ++k) G[a][b] += A[k * 9 + a] * A[k * 9 + b];
    for (int j = 0; j < 9; ++j) {
      double d = G[j][j];
      for (int k = 0; k < j; ++k) d -= Lc[j][k] * Lc[j][k];
      if (!(d > 0)) return false;
      Lc[j][j] = std::sqrt(d);
      for (int i = j + 1; i < 9; ++i) {
        double v = G[i][j];
        for (int k = 0; k < j; ++k) v -= Lc[i][k] * Lc[j][k];
        Lc[i][j] = v / Lc[j][j];
      }
    }
    for (int j = 0; j < 9; ++j) {  // W = L^{-1}, column by column
      Wm[j][j] = 1.0 / Lc[j][j];
      for (int i = j + 1; i < 9; ++i) {
        double v = 0;
        for (int k = j; k < i; ++k) v -= Lc[i][k] * Wm[k][j];
        Wm[i][j] = v / Lc[i][i];
      }
    }
    double pmax = 0, dmax = 0;
    for (int d = 0; d < 9; ++d)
      for (int k = 0; k < K; ++k) {
        double s = 0;  // (W^T W A^T)[d][k]
        for (int i = 0; i < 9; ++i) {
          double wa = 0;
          for (int j = 0; j <= i; ++j) wa += Wm[i][j] * A[k * 9 + j];
          s += Wm[i][d] * wa;
        }
        pmax = std::max(pmax, std::fabs(P[d * K + k]));
        dmax = std::max(dmax, std::fabs(s - P[d * K + k]));
      }
    if (!(dmax <= 1e-9 * pmax)) return false;
    for (int i = 0, e = 0; i < 9; ++i)
      for (int j = 0; j <= i; ++j) op[e++] = Wm[i][j];
  }
#else
  for (int d = 0; d < 9; ++d)
    for (int k = 0; k < K; ++k) op[d * L.K + k] = P[d * K + k] / (d < 3 ? h : h * h);
#endif
  const int8_t* ss = &gm.sub_slot[i * L.M * L.NM];
  // a tet of a hybrid mesh has 4 of the layout's 6 sub-stencils (the rest stay 0)
  const int Mi = gm.type[i] == 4 ? 4 : L.M;
  for (int m = 0; m < Mi; ++m) {
    int n = 0;
    double As[3 * 8];
    int slots[8];
    for (int j = 0; j < L.NM; ++j)
      if (ss[m * L.NM + j] >= 0) {
        slots[n] = ss[m * L.NM + j];
        for (int a = 0; a < 3; ++a) As[n * 3 + a] = A[slots[n] * 9 + a];
        ++n;
      }
    double Ps[3 * 8];
    if (n < 3 || !pinv_qr(n, 3, As, Ps)) return false;
    double* om = op + L.op0_entries() + m * 3 * L.NM;
    for (int d = 0; d < 3; ++d)
      for (int j = 0; j < n; ++j) om[d * L.NM + j] = Ps[d * n + j] / h;
  }
  return true;
}

RankPlan build_rank_plan(const GlobalMesh& gm, int rank) {
  const Layout& L = gm.lay;
  const int64_t nc = gm.nc;
  RankPlan rp;
  PhaseTimer pt("rank plan");
  rp.rank = rank;
  std::vector<int64_t> owned;
  for (int64_t i = 0; i < nc; ++i)
    if (gm.part[i] == rank) owned.push_back(i);
  if (owned.empty()) throw Error(1, "rank " + std::to_string(rank) + " owns no cells");
  if (gm.only_rank >= 0 && rank != gm.only_rank)
    throw Error(1, "this mesh holds rank " + std::to_string(gm.only_rank) + "'s region only");
  // Morton order over the global bounding box of centroids
  const double* lo = gm.bbox_lo;
  const double* hi = gm.bbox_hi;
  auto morton = [&](int64_t i) {
    uint64_t k = 0;
    for (int a = 0; a < 3; ++a) {
      double s = hi[a] > lo[a] ? (gm.C[3 * i + a] - lo[a]) / (hi[a] - lo[a]) : 0.0;
      uint64_t q = (uint64_t)std::min(2097151.0, std::max(0.0, s * 2097151.0));
      k |= spread21(q) << a;
    }
    return k;
  };
  std::vector<uint64_t> mk(nc);
  for (int64_t i = 0; i < nc; ++i) mk[i] = morton(i);
  auto by_morton = [&](int64_t a, int64_t b) { return mk[a] != mk[b] ? mk[a] < mk[b] : a < b; };
  std::sort(owned.begin(), owned.end(), by_morton);
  rp.n_owned = (int64_t)owned.size();
  // ghost layers by face adjacency (BC ghosts excluded)
  std::vector<int8_t> layer(nc, -1);  // 0 owned, 1..3 ghost layers
  for (int64_t i : owned) layer[i] = 0;
  std::vector<int64_t> frontier = owned;
  std::vector<std::vector<int64_t>> ghosts(3);
  for (int l = 1; l <= 3 && gm.n_ranks > 1; ++l) {
    std::vector<int64_t> next;
    for (int64_t i : frontier)
      for (int p = 0; p < L.nfaces; ++p) {
        int64_t j = gm.nbr_id[i * 6 + p];
        if (j >= 0 && j < nc && layer[j] < 0) {
          layer[j] = (int8_t)l;
          next.push_back(j);
        }
      }
    ghosts[l - 1] = next;
    rp.ghost_layer[l - 1] = (int64_t)next.size();
    frontier.swap(next);
  }
  // partition ghosts grouped by owner rank, then layer, then global id
  std::vector<int64_t> pg;
  for (auto& g : ghosts) pg.insert(pg.end(), g.begin(), g.end());
  std::sort(pg.begin(), pg.end(), [&](int64_t a, int64_t b) {
    if (gm.part[a] != gm.part[b]) return gm.part[a] < gm.part[b];
    return a < b;  // global-id order == the owner's send order
  });
  rp.n_pghost = (int64_t)pg.size();
  rp.l2g = owned;
  rp.l2g.insert(rp.l2g.end(), pg.begin(), pg.end());
  std::vector<int32_t> g2l(nc, -1);  // global cell -> local id (-1: not on this rank)
  for (size_t k = 0; k < rp.l2g.size(); ++k) g2l[rp.l2g[k]] = (int32_t)k;
  pt.lap("morton + ghost layers");
  // Reconstruction order (P:856-866 overlap): [early | pad | late | L1 ghosts], where
  // "early" owned cells have stencils made of owned cells and of boundary ghosts of
  // owned cells only, so they are reconstructed while the halo exchange is in
  // flight; the early block is padded (recon_cell = -1) to a whole 128-cell tile.
  std::vector<char> early_cell(rp.n_owned, 0);
  {
    std::vector<int32_t> early, late;
    for (int64_t i = 0; i < rp.n_owned; ++i) {
      const int64_t gi = owned[i];
      bool e = true;
      for (int64_t o = gm.big_off[gi]; o < gm.big_off[gi + 1] && e; ++o) {
        const int64_t id = gm.big_id[o];
        const int64_t owner_cell = id < nc ? id : gm.g_cell[id - nc];
        e = gm.part[owner_cell] == rank;
      }
      early_cell[i] = e;
      (e ? early : late).push_back((int32_t)i);
    }
    rp.n_recon_early = (int64_t)early.size();
    rp.recon_cell = early;
    rp.recon_cell.resize((early.size() + 127) / 128 * 128, -1);
    rp.recon_late0 = (int64_t)rp.recon_cell.size();
    rp.recon_cell.insert(rp.recon_cell.end(), late.begin(), late.end());
    const size_t g0 = rp.recon_cell.size();
    for (int64_t g : pg)
      if (layer[g] == 1) rp.recon_cell.push_back(g2l[g]);
    // layer-1 ghosts in Morton order too, so their reconstruction tiles stay compact
    std::sort(rp.recon_cell.begin() + g0, rp.recon_cell.end(),
              [&](int32_t a, int32_t b) { return by_morton(rp.l2g[a], rp.l2g[b]); });
  }
  rp.n_recon = (int64_t)rp.recon_cell.size();
  pt.lap("recon order");
  // BC ghosts needed: those of faces of recon cells and of their neighbours
  std::vector<int32_t> bg2l(gm.g_cell.size(), -1);  // boundary ghost -> local id
  std::vector<int64_t> bg_used;                      // boundary ghosts in local order
  auto local_of = [&](int64_t id) -> int32_t {
    if (id < nc) {
      if (g2l[id] < 0) throw Error(1, "ghost closure violated for cell " + std::to_string(id));
      return g2l[id];
    }
    const int64_t g = id - nc;
    if (bg2l[g] >= 0) return bg2l[g];
    int32_t l = (int32_t)(rp.n_owned + rp.n_pghost + (int64_t)bg_used.size());
    bg2l[g] = l;
    bg_used.push_back(g);
    rp.bg_cell.push_back(-1);  // resolved below
    rp.bg_bc.push_back(gm.g_bc[g]);
    rp.bg_normal.push_back(gm.g_normal[3 * g]);
    rp.bg_normal.push_back(gm.g_normal[3 * g + 1]);
    rp.bg_normal.push_back(gm.g_normal[3 * g + 2]);
    return l;
  };
  const int K = L.K, M = L.M, NM = L.NM, E = L.op_entries();
  const int64_t Rn = rp.n_recon;
  // entry-major arrays use a stride padded to the 64-cell tile so every
  // per-tile operator row is one aligned 512-byte bulk copy
  const int64_t R = (Rn + 127) / 128 * 128;
  rp.ld = R;
  rp.st_id.assign((size_t)K * R, 0);
  rp.sub_slot.assign((size_t)M * NM * R, 0);
  rp.st_shift.assign((size_t)K * R, 13);
  rp.op.assign((size_t)E * R, 0.0);
  rp.geo.assign((size_t)8 * R, 0.0);
  if (L.cell_type == 6) rp.n_sub.assign((size_t)R, 6);
  // tiled entry-major layout: entry e of cell r at ((r/128)*NE + e)*128 + r%128, so one
  // 128-cell block reads its operators from one contiguous range (DRAM page locality)
  auto ti = [](int64_t r, int ne, int e) { return (size_t)(((r >> 7) * ne + e) << 7) + (size_t)(r & 127); };
  // operators: tiled by entry PAIRS, so one 16-byte load gives a cell two consecutive
  // entries (a warp load = 512 contiguous bytes); E is even (K even, 3*M*NM even)
  auto tp = [](int64_t r, int ne, int e) {
    return (((size_t)((r >> 7) * (ne / 2) + (e >> 1)) << 7 | (size_t)(r & 127)) << 1) | (size_t)(e & 1);
  };
  rp.st_id_tiled.assign((size_t)K * R, 0);
  // boundary ghosts met in stencils get their local ids first (serial, in
  // reconstruction order), so the per-cell fill below only reads the maps
  for (int64_t r = 0; r < Rn; ++r) {
    if (rp.recon_cell[r] < 0) continue;
    const int64_t gi = rp.l2g[rp.recon_cell[r]];
    for (int64_t o = gm.big_off[gi]; o < gm.big_off[gi + 1]; ++o)
      if (gm.big_id[o] >= nc) local_of(gm.big_id[o]);
  }
  int smin = 1 << 30, smax = 0;
  int64_t bad = -1, lsq_bad = -1;
#pragma omp parallel for schedule(static) reduction(min : smin) reduction(max : smax)
  for (int64_t r = 0; r < Rn; ++r) {
    if (rp.recon_cell[r] < 0) continue;  // padding of the early block
    int64_t gi = rp.l2g[rp.recon_cell[r]];
    int64_t o0 = gm.big_off[gi];
    int kk = (int)(gm.big_off[gi + 1] - o0);
    if (rp.recon_cell[r] < rp.n_owned) {
      smin = std::min(smin, kk);
      smax = std::max(smax, kk);
    }
    for (int k = 0; k < K; ++k) {
      int32_t l = rp.recon_cell[r];
      if (k < kk) {
        const int64_t id = gm.big_id[o0 + k];
        l = id < nc ? g2l[id] : bg2l[id - nc];
        if (l < 0) {
#pragma omp critical
          bad = id;
          l = 0;
        }
      }
      rp.st_id[(size_t)k * R + r] = l;
      rp.st_id_tiled[ti(r, K, k)] = l;
    }
    for (int s = 0; s < M * NM; ++s) {
      int8_t v = gm.sub_slot[gi * M * NM + s];
      rp.sub_slot[ti(r, M * NM, s)] = (uint8_t)(v < 0 ? 0 : v);
    }
    if (L.cell_type == 6) rp.n_sub[r] = (uint8_t)(gm.type[gi] == 4 ? 4 : 6);
    // streaming order of the operator entries (hot.cuh k_recon): A0+ member-major
    // (row k*9 + d), then the sub-stencil operators (row 9K + (m*NM + j)*3 + d)
    double op[9 * 64 + 8 * 3 * 8] = {};
    if (!cell_operators(gm, gi, op)) {
#pragma omp critical
      if (lsq_bad < 0 || gi < lsq_bad) lsq_bad = gi;
    }
    const int E0 = L.op0_entries();
#if HGKS_RECON_NE
    for (int e = 0; e < E0; ++e) rp.op[tp(r, E, e)] = op[e];
    for (int k = 0; k < K; ++k) {  // periodic image of member k: shift / box length per axis in {-1, 0, 1}
      int code = 13;
      if (k < kk) {
        code = 0;
        for (int a = 2; a >= 0; --a) {
          const double sh = gm.big_shift[3 * (o0 + k) + a];
          const int sa = gm.per_len[a] > 0 ? (int)std::lround(sh / gm.per_len[a]) : 0;
          if (sa < -1 || sa > 1) {
#pragma omp critical
            lsq_bad = gi;
          }
          code = 3 * code + (sa + 1);
        }
      }
      rp.st_shift[ti(r, K, k)] = (uint8_t)code;
    }
#else
    for (int d = 0; d < 9; ++d)
      for (int k = 0; k < K; ++k) rp.op[tp(r, E, k * 9 + d)] = op[d * K + k];
#endif
    for (int m = 0; m < M; ++m)
      for (int d = 0; d < 3; ++d)
        for (int j = 0; j < NM; ++j) rp.op[tp(r, E, E0 + (m * NM + j) * 3 + d)] = op[E0 + (m * 3 + d) * NM + j];
    double V = gm.V[gi];
    rp.geo[ti(r, 8, 0)] = std::pow(V, 2.0 / 3.0);
    rp.geo[ti(r, 8, 1)] = std::pow(V, 4.0 / 3.0);
    for (int k = 0; k < 6; ++k) rp.geo[ti(r, 8, 2 + k)] = gm.M2[6 * gi + k];
  }
  if (bad >= 0) throw Error(1, "ghost closure violated for cell " + std::to_string(bad));
  if (lsq_bad >= 0) throw Error(3, "rank-deficient least-squares stencil at cell " + std::to_string(lsq_bad));
  rp.stencil_min = smin;
  rp.stencil_max = smax;
  pt.lap("tiled per-cell arrays");
  // faces computed by this rank: every face of an owned cell
  std::vector<int64_t> fl;
  {
    std::vector<char> seen(gm.nf, 0);
    for (int64_t i : owned)
      for (int p = 0; p < L.nfaces; ++p) {
        int64_t f = gm.cell_face[i * 6 + p];
        if (f >= 0 && !seen[f]) {
          seen[f] = 1;
          fl.push_back(f);
        }
      }
  }
  for (int64_t f : fl)
    if (gm.f_nb[f] < 0) local_of(nc + gm.f_ghost[f]);
  // order: triangles before quadrilaterals (one flux instantiation per face kind), then
  // early interior faces (both cells reconstructed before the exchange completes), late
  // interior faces, wall, farfield; by min local endpoint within
  auto is_early = [&](int64_t gcell) {
    const int32_t l = g2l[gcell];
    return l < rp.n_owned && early_cell[l];
  };
  auto fkey = [&](int64_t f) -> std::pair<int, int64_t> {
    int cls = gm.f_nb[f] >= 0 ? (is_early(gm.f_owner[f]) && is_early(gm.f_nb[f]) ? 0 : 1)
                              : (gm.f_bc[f] == 1 ? 2 : 3);
    int64_t a = g2l[gm.f_owner[f]];
    int64_t b = gm.f_nb[f] >= 0 ? g2l[gm.f_nb[f]] : a;
    return {(gm.f_nv[f] == 4 ? 4 : 0) + cls, std::min(a, b)};
  };
  {
    // sort keys computed once: (class, min local endpoint, position) = a stable sort
    std::vector<std::pair<std::pair<int, int64_t>, int64_t>> keyed(fl.size());
    for (size_t k = 0; k < fl.size(); ++k) keyed[k] = {fkey(fl[k]), (int64_t)k};
    std::sort(keyed.begin(), keyed.end());
    std::vector<int64_t> sorted(fl.size());
    for (size_t k = 0; k < fl.size(); ++k) sorted[k] = fl[keyed[k].second];
    fl.swap(sorted);
  }
  rp.n_faces = (int64_t)fl.size();
  for (int64_t f : fl) {
    const int kc = fkey(f).first, k = kc >> 2, cls = kc & 3;
    FaceClass& F = rp.fcls[k];
    if (cls == 0) ++F.n_if_early;
    if (cls <= 1) ++F.n_if;
    else if (cls == 2) ++F.n_wf;
    else ++F.n_ff;
  }
  rp.fcls[1].base = rp.fcls[0].n_if + rp.fcls[0].n_wf + rp.fcls[0].n_ff;
  for (const FaceClass& F : rp.fcls) {
    rp.n_if_early += F.n_if_early;
    rp.n_if += F.n_if;
    rp.n_wf += F.n_wf;
    rp.n_ff += F.n_ff;
  }
  pt.lap("face list + order");
  rp.f_geo_stride = 3 * L.nv + 3;
  rp.f_cells.resize(2 * rp.n_faces);
  rp.f_geo.assign((size_t)rp.f_geo_stride * rp.n_faces, 0.0);
  std::vector<int32_t> f2l(gm.nf, -1);  // global face -> local face id
  for (int64_t k = 0; k < rp.n_faces; ++k) {
    int64_t f = fl[k];
    f2l[f] = (int32_t)k;
    int64_t o = gm.f_owner[f];
    rp.f_cells[2 * k] = g2l[o];
    rp.f_cells[2 * k + 1] = gm.f_nb[f] >= 0 ? g2l[gm.f_nb[f]] : local_of(nc + gm.f_ghost[f]);
    double* fg = &rp.f_geo[(size_t)rp.f_geo_stride * k];
    const int nv = gm.f_nv[f];
    for (int q = 0; q < nv; ++q)
      for (int a = 0; a < 3; ++a) fg[3 * q + a] = gm.f_vert[12 * f + 3 * q + a] - gm.C[3 * o + a];
    // d = c_owner - (c_nb + shift): the neighbour evaluates at r_l + d
    if (gm.f_nb[f] >= 0)
      for (int a = 0; a < 3; ++a) fg[3 * nv + a] = gm.C[3 * o + a] - (gm.C[3 * gm.f_nb[f] + a] + gm.f_shift[3 * f + a]);
  }
  pt.lap("face arrays");
  // update arrays
  rp.cf.assign((size_t)L.nfaces * rp.n_owned, 0);
  rp.inv_v.resize(rp.n_owned);
  rp.h_dt.resize(rp.n_owned);
  for (int64_t r = 0; r < rp.n_owned; ++r) {
    int64_t gi = owned[r];
    for (int p = 0; p < L.nfaces; ++p) {
      int64_t f = gm.cell_face[gi * 6 + p];
      if (f < 0) {  // no face p (a tet of a hybrid mesh): the zero row past the last face
        rp.cf[(size_t)p * rp.n_owned + r] = (int32_t)rp.n_faces;
        continue;
      }
      int32_t lf = f2l[f];
      rp.cf[(size_t)p * rp.n_owned + r] = gm.f_owner[f] == gi ? lf : ~lf;
    }
    rp.inv_v[r] = 1.0 / gm.V[gi];
    rp.h_dt[r] = gm.h_dt[gi];
  }
  // resolve BC ghost interior cells (must be local)
  for (size_t k = 0; k < bg_used.size(); ++k) rp.bg_cell[k] = local_of(gm.g_cell[bg_used[k]]);
  rp.n_bghost = (int64_t)bg_used.size();
#if HGKS_RECON_NE
  // centroid and second moments of every local row (members of the rebuilt LSQ rows)
  rp.cgeo.assign((size_t)10 * rp.n_local(), 0.0);
  for (int64_t l = 0; l < rp.n_local(); ++l) {
    const double *c, *m2;
    if (l < rp.n_owned + rp.n_pghost) {
      const int64_t gi = rp.l2g[l];
      c = &gm.C[3 * gi];
      m2 = &gm.M2[6 * gi];
    } else {
      const int64_t g = bg_used[l - rp.n_owned - rp.n_pghost];
      c = &gm.gC[3 * g];
      m2 = &gm.gM2[6 * g];
    }
    for (int a = 0; a < 3; ++a) rp.cgeo[10 * l + a] = c[a];
    for (int a = 0; a < 6; ++a) rp.cgeo[10 * l + 3 + a] = m2[a];
  }
#endif
  // exchange plan: peers = owner ranks of my ghosts, and ranks that ghost my cells
  if (gm.n_ranks > 1) {
    std::vector<std::vector<int32_t>> sends(gm.n_ranks);
    // cells I own that appear in another rank's 3-layer closure
    std::vector<std::vector<char>> want(gm.n_ranks);
    for (int q = 0; q < gm.n_ranks; ++q) {
      if (q == rank) continue;
      // BFS from q's owned cells, 3 layers
      std::vector<int8_t> lay(nc, -1);
      std::vector<int64_t> fr;
      for (int64_t i = 0; i < nc; ++i)
        if (gm.part[i] == q) {
          lay[i] = 0;
          fr.push_back(i);
        }
      for (int l = 1; l <= 3; ++l) {
        std::vector<int64_t> nx;
        for (int64_t i : fr)
          for (int p = 0; p < L.nfaces; ++p) {
            int64_t j = gm.nbr_id[i * 6 + p];
            if (j >= 0 && j < nc && lay[j] < 0) {
              lay[j] = (int8_t)l;
              nx.push_back(j);
            }
          }
        fr.swap(nx);
      }
      std::vector<int64_t> mine;
      for (int64_t i = 0; i < nc; ++i)
        if (lay[i] > 0 && gm.part[i] == rank) mine.push_back(i);
      std::sort(mine.begin(), mine.end());
      for (int64_t i : mine) sends[q].push_back(g2l[i]);
    }
    for (int q = 0; q < gm.n_ranks; ++q) {
      if (q == rank) continue;
      int64_t off = -1, cnt = 0;
      for (int64_t k = 0; k < rp.n_pghost; ++k)
        if (gm.part[pg[k]] == q) {
          if (off < 0) off = rp.n_owned + k;
          ++cnt;
        }
      if (cnt == 0 && sends[q].empty()) continue;
      rp.peers.push_back(q);
      rp.send_off.push_back((int64_t)rp.send_list.size());
      rp.send_cnt.push_back((int64_t)sends[q].size());
      rp.send_list.insert(rp.send_list.end(), sends[q].begin(), sends[q].end());
      rp.recv_off.push_back(off < 0 ? rp.n_owned : off);
      rp.recv_cnt.push_back(cnt);
    }
  }
  // faces of owned cells whose other side another rank owns (this rank's share of the cut)
  for (int64_t r = 0; r < rp.n_owned; ++r)
    for (int p = 0; p < L.nfaces; ++p) {
      const int64_t j = gm.nbr_id[owned[r] * 6 + p];
      if (j >= 0 && j < nc && gm.part[j] != rank) ++rp.rank_cut_faces;
    }
  // region builds index cells by position in the region: report global ids
  if (!gm.gid.empty())
    for (auto& id : rp.l2g) id = gm.gid[id];
  pt.lap("update arrays, plans");
  return rp;
}

}  // namespace hgks
