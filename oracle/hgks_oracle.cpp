// ============================================================================
// HGKS CPU ORACLE  --  TEST INFRASTRUCTURE ONLY
// ============================================================================
// Plain, slow, scalar fp64 implementation of the high-order gas-kinetic scheme
// of Wang, Cao & Pan (arXiv 2407.00656, /root/reference/PAPER.md, cited "P:n").
// It is the correctness authority for the CUDA path in paper_2407_00656_b200/.
//
//  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
//    --impl reference legs may load this library.  The product never does.
//  * It shares NO code with the product (no headers, helpers or tables): it
//    builds its own connectivity, geometry and least-squares systems from the
//    same input arrays (paper_2407_00656_b200/workloads.py).
//  * Every step follows the paper's order and notation; where the paper is
//    silent the reading is the one listed in DESIGN.md ("Readings", R1-R26,
//    which restate SURVEY.md 8(c) Q1-Q26).  Differences from the CUDA path are
//    deliberate: LSQ by Householder QR at every stage (no stored operators),
//    Eq. (weno) evaluated literally at each Gauss point (no collapse), the
//    smoothness indicator by exact cell quadrature (no closed form), and the
//    kinetic flux from generic polynomial moment sums (no unrolled algebra).
//
// Parity pins (tests/test_oracle_*.py): geometry closure and volumes,
// depth-2 BFS stencils, LSQ exactness, beta closed values, moments vs
// numerical quadrature, slopes vs numpy solve, single-face flux vs brute-force
// velocity/time quadrature of Eq. (flux), tau=0 Euler-chain identity,
// S2O4 Taylor polynomial, conservation, free-stream preservation, and the
// paper's Table 3 convergence (T3), the farfield Riemann state against the
// characteristic conditions, and the wall mirror (R25) on a walled box: no mass
// or energy through the wall at tau = 0 and the closed-form no-slip stagnation
// pressure (tests/test_oracle_wall.py).
// ============================================================================
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

using Vec3 = std::array<double, 3>;
using Mat3 = std::array<std::array<double, 3>, 3>;

constexpr int kTet = 4, kPrism = 6, kHex = 8;
constexpr int kWall = 1, kFarfield = 2;

Vec3 sub(const Vec3& a, const Vec3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
Vec3 add(const Vec3& a, const Vec3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
Vec3 scale(const Vec3& a, double s) { return {a[0] * s, a[1] * s, a[2] * s}; }
double dot(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }

struct OracleError : std::runtime_error {
  int code;
  OracleError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum { E_OK = 0, E_ARG = 1, E_MESH = 2, E_STENCIL = 3, E_POSITIVITY = 6, E_STATE = 7 };

// ---------------------------------------------------------------------------
// Configuration (readings R4, R6, R7, R13, R14, R24)
// ---------------------------------------------------------------------------
struct Config {
  double gamma = 1.4;
  double cfl = 0.3;
  double fixed_dt = 0.0;   // > 0 overrides the CFL rule
  int tau_mode = 0;        // 0: tau = 0; 1: tau = mu/p + C1|pl-pr|/(pl+pr) dt
  double c1 = 1.0;
  double mu_inf = 0.0, t_inf = 1.0, mu_exp = 0.7;  // mu = mu_inf (T/T_inf)^0.7
  double eps = 1e-10;      // epsilon of the WENO weights (R14)
  int omega_pow = 1;       // exponent of tau_Z/(beta+eps) (R13)
  double fs[5] = {1.0, 0.0, 0.0, 0.0, 1.0 / 1.4};  // free stream rho, U, V, W, p
  int dq0_mode = 0;        // equilibrium slopes dQ0 (P:306-308 gives only <a-bar> = dQ0/dn):
                           // 0 average of the two reconstructed gradients (R9), 1 kinetic weighting
                           // (R9k), 2 linear-weight (gamma) recombination averaged (R9s)
  double prandtl = 1.0;    // Pr; != 1: heat-flux (Prandtl-number) correction of the energy flux (R29)
  double K() const { return (5.0 - 3.0 * gamma) / (gamma - 1.0); }
};

// ---------------------------------------------------------------------------
// O1 Geometry
// ---------------------------------------------------------------------------
// Local faces: tet face p is opposite local node p; hex faces in
// VTK/Gmsh node order, 0 and 5 the opposed pair, 1..4 a ring (R17).
const int kTetFace[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
const int kHexFace[6][4] = {{0, 1, 2, 3}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}, {4, 5, 6, 7}};
// Triangular prism (VTK wedge order, reading R30): faces 0 / 1 the two triangles, 2..4 the
// quadrilateral sides in ring order (side p joins triangle edges (p-2, p-1 mod 3)).
const int kPrismFace[5][4] = {{0, 1, 2, -1}, {3, 4, 5, -1}, {0, 1, 4, 3}, {1, 2, 5, 4}, {2, 0, 3, 5}};

struct CellGeom {
  double V = 0;
  Vec3 c{};
  double M2[3][3] = {};  // mean over the cell of (x-c)(x-c)^T
};

// Reference points of the trilinear hex on [0,1]^3 (VTK order)
const double kHexRef[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

void gauss3(double* x, double* w) {  // 3-point Gauss-Legendre on [0,1]
  const double s = std::sqrt(0.6);
  x[0] = 0.5 * (1 - s); x[1] = 0.5; x[2] = 0.5 * (1 + s);
  w[0] = 5.0 / 18; w[1] = 8.0 / 18; w[2] = 5.0 / 18;
}

// Quadrature points (physical) and weights (summing to the cell volume) exact
// for polynomials of degree <= 2 on tets and for (degree-2 poly)*|J| on
// trilinear hexes.  Used for geometry moments and for beta.
void cell_quadrature(int type, const std::vector<Vec3>& v, std::vector<Vec3>& pts, std::vector<double>& wts) {
  pts.clear(); wts.clear();
  if (type == kTet) {
    Vec3 e1 = sub(v[1], v[0]), e2 = sub(v[2], v[0]), e3 = sub(v[3], v[0]);
    double V = std::fabs(dot(e1, cross(e2, e3))) / 6.0;
    const double a = 0.5854101966249685, b = 0.1381966011250105;  // degree-2 4-point rule
    for (int q = 0; q < 4; ++q) {
      double lam[4] = {b, b, b, b};
      lam[q] = a;
      Vec3 x{0, 0, 0};
      for (int k = 0; k < 4; ++k) x = add(x, scale(v[k], lam[k]));
      pts.push_back(x);
      wts.push_back(V / 4.0);
    }
  } else if (type == kPrism) {
    // wedge map X = sum_a N_a v_a, N = (1-xi-eta, xi, eta) x (1-zeta, zeta): |J| is linear in
    // (xi, eta) and quadratic in zeta, so Radon's 7-point degree-5 triangle rule x 3-point
    // Gauss in zeta integrates (degree-2 poly) * |J| exactly
    const double r15 = std::sqrt(15.0);
    const double a1 = (9 - 2 * r15) / 21, b1 = (6 + r15) / 21, a2 = (9 + 2 * r15) / 21, b2 = (6 - r15) / 21;
    const double w0 = 9.0 / 80, w1 = (155 + r15) / 2400, w2 = (155 - r15) / 2400;  // sum 1/2
    const double tri[7][3] = {{1.0 / 3, 1.0 / 3, w0}, {a1, b1, w1}, {b1, a1, w1}, {b1, b1, w1},
                              {a2, b2, w2}, {b2, a2, w2}, {b2, b2, w2}};
    double g[3], gw[3];
    gauss3(g, gw);
    for (int q = 0; q < 7; ++q)
      for (int k = 0; k < 3; ++k) {
        const double xi = tri[q][0], et = tri[q][1], ze = g[k];
        const double L[3] = {1 - xi - et, xi, et};
        Vec3 X{0, 0, 0}, dxi{0, 0, 0}, det_{0, 0, 0}, dze{0, 0, 0};
        for (int a = 0; a < 3; ++a) {
          X = add(X, add(scale(v[a], L[a] * (1 - ze)), scale(v[a + 3], L[a] * ze)));
          dze = add(dze, scale(sub(v[a + 3], v[a]), L[a]));
        }
        // d/dxi: L = (1-xi-eta, xi, eta) -> (-1, 1, 0); d/deta -> (-1, 0, 1)
        const Vec3 b0 = add(scale(v[0], 1 - ze), scale(v[3], ze)), b1v = add(scale(v[1], 1 - ze), scale(v[4], ze)),
                   b2v = add(scale(v[2], 1 - ze), scale(v[5], ze));
        dxi = sub(b1v, b0);
        det_ = sub(b2v, b0);
        const double J = std::fabs(dot(dxi, cross(det_, dze)));
        pts.push_back(X);
        wts.push_back(tri[q][2] * gw[k] * J);
      }
  } else {
    double g[3], gw[3];
    gauss3(g, gw);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) {
          double xi = g[i], et = g[j], ze = g[k];
          Vec3 X{0, 0, 0}, dxi{0, 0, 0}, det_{0, 0, 0}, dze{0, 0, 0};
          for (int a = 0; a < 8; ++a) {
            double rx = kHexRef[a][0], ry = kHexRef[a][1], rz = kHexRef[a][2];
            double fx = rx ? xi : 1 - xi, fy = ry ? et : 1 - et, fz = rz ? ze : 1 - ze;
            double sx = rx ? 1 : -1, sy = ry ? 1 : -1, sz = rz ? 1 : -1;
            X = add(X, scale(v[a], fx * fy * fz));
            dxi = add(dxi, scale(v[a], sx * fy * fz));
            det_ = add(det_, scale(v[a], fx * sy * fz));
            dze = add(dze, scale(v[a], fx * fy * sz));
          }
          double J = std::fabs(dot(dxi, cross(det_, dze)));
          pts.push_back(X);
          wts.push_back(gw[i] * gw[j] * gw[k] * J);
        }
  }
}

CellGeom cell_geometry(int type, const std::vector<Vec3>& v) {
  CellGeom g;
  if (type == kTet) {
    // V = |det|/6, centroid = vertex mean, M2 = (1/20) sum d d^T (exact for tets)
    Vec3 e1 = sub(v[1], v[0]), e2 = sub(v[2], v[0]), e3 = sub(v[3], v[0]);
    g.V = std::fabs(dot(e1, cross(e2, e3))) / 6.0;
    g.c = {0, 0, 0};
    for (int k = 0; k < 4; ++k) g.c = add(g.c, scale(v[k], 0.25));
    for (int k = 0; k < 4; ++k) {
      Vec3 d = sub(v[k], g.c);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g.M2[a][b] += d[a] * d[b] / 20.0;
    }
  } else {
    std::vector<Vec3> pts;
    std::vector<double> w;
    cell_quadrature(type, v, pts, w);
    g.V = 0;
    g.c = {0, 0, 0};
    for (size_t q = 0; q < pts.size(); ++q) { g.V += w[q]; g.c = add(g.c, scale(pts[q], w[q])); }
    g.c = scale(g.c, 1.0 / g.V);
    for (size_t q = 0; q < pts.size(); ++q) {
      Vec3 d = sub(pts[q], g.c);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g.M2[a][b] += w[q] * d[a] * d[b] / g.V;
    }
  }
  return g;
}

struct GaussPoint {
  Vec3 x{};     // position (owner's coordinates)
  Vec3 n{};     // unit normal out of the owner ("local normal direction")
  double wS = 0;  // omega_G * S
};

// Face Gauss points (R10): triangle 3-point degree-2 rule (barycentric
// 2/3,1/6,1/6), quad 2x2 Gauss-Legendre on the bilinear surface with per-GP
// normal and weight*area = |X_xi x X_eta|/4.
std::vector<GaussPoint> face_gauss_points(const std::vector<Vec3>& p) {
  std::vector<GaussPoint> gp;
  if (p.size() == 3) {
    Vec3 nn = cross(sub(p[1], p[0]), sub(p[2], p[0]));
    double area = 0.5 * norm(nn);
    Vec3 n = scale(nn, 1.0 / norm(nn));
    for (int k = 0; k < 3; ++k) {
      double lam[3] = {1.0 / 6, 1.0 / 6, 1.0 / 6};
      lam[k] = 2.0 / 3;
      GaussPoint g;
      g.x = add(add(scale(p[0], lam[0]), scale(p[1], lam[1])), scale(p[2], lam[2]));
      g.n = n;
      g.wS = area / 3.0;
      gp.push_back(g);
    }
  } else {
    const double r = 0.5 / std::sqrt(3.0);
    const double q[2] = {0.5 - r, 0.5 + r};
    for (int b = 0; b < 2; ++b)
      for (int a = 0; a < 2; ++a) {
        double xi = q[a], et = q[b];
        Vec3 X = add(add(scale(p[0], (1 - xi) * (1 - et)), scale(p[1], xi * (1 - et))),
                     add(scale(p[2], xi * et), scale(p[3], (1 - xi) * et)));
        Vec3 Xxi = add(scale(sub(p[1], p[0]), 1 - et), scale(sub(p[2], p[3]), et));
        Vec3 Xet = add(scale(sub(p[3], p[0]), 1 - xi), scale(sub(p[2], p[1]), xi));
        Vec3 nn = cross(Xxi, Xet);
        GaussPoint g;
        g.x = X;
        g.n = scale(nn, 1.0 / norm(nn));
        g.wS = 0.25 * norm(nn);
        gp.push_back(g);
      }
  }
  return gp;
}

// ---------------------------------------------------------------------------
// O2/O3 Mesh, connectivity, Alg. 1, stencils
// ---------------------------------------------------------------------------
struct Face {
  int owner = -1;    // lower input cell id (R19)
  int nb = -1;       // neighbour cell id, or -1 for a physical boundary face
  int bc = 0;        // boundary tag for nb == -1
  int ghost = -1;    // ghost index for boundary faces
  Vec3 shift{0, 0, 0};  // neighbour image = neighbour cell translated by shift (R23)
  std::vector<GaussPoint> gp;
  double area = 0;
};

struct Member {  // a stencil member: cell id (ghosts: n_cells + g) and periodic shift
  int id;
  Vec3 s;
};

struct Mesh {
  int n_cells = 0, n_ghosts = 0;
  std::vector<int> type;
  std::vector<std::vector<Vec3>> cell_xyz;
  std::vector<CellGeom> geom;               // [n_cells + n_ghosts]
  std::vector<Face> faces;
  std::vector<std::vector<int>> cell_face;  // local face order
  std::vector<std::vector<Member>> neighbor;  // CellNeighbor: one entry per local face
  std::vector<std::vector<Member>> big;       // S_i^WENO \ {i} (Alg. 1 order, R18)
  std::vector<std::vector<std::vector<Member>>> subs;  // S_{i_m}^WENO \ {i}
  std::vector<int> ghost_cell, ghost_face, ghost_bc;   // per ghost
  std::vector<double> h_dt;  // V_i / max_p S_ip (R6)
};

int n_faces_of(int t) { return t == kTet ? 4 : (t == kPrism ? 5 : 6); }

std::vector<int> face_local_nodes(int t, int p) {
  if (t == kTet) return {kTetFace[p][0], kTetFace[p][1], kTetFace[p][2]};
  if (t == kPrism) {
    if (p < 2) return {kPrismFace[p][0], kPrismFace[p][1], kPrismFace[p][2]};
    return {kPrismFace[p][0], kPrismFace[p][1], kPrismFace[p][2], kPrismFace[p][3]};
  }
  return {kHexFace[p][0], kHexFace[p][1], kHexFace[p][2], kHexFace[p][3]};
}

struct MeshInputC {
  const double* xyz; int64_t n_nodes;
  const int8_t* type; const int64_t* cell_nodes; int64_t n_cells;
  const double* per_origin; const double* per_len;
  const int64_t* bface_nodes; const int32_t* bface_tag; int64_t n_bf;
};

Mesh build_mesh(const MeshInputC& in) {
  Mesh m;
  m.n_cells = (int)in.n_cells;
  m.type.resize(m.n_cells);
  m.cell_xyz.resize(m.n_cells);
  for (int i = 0; i < m.n_cells; ++i) {
    int t = in.type[i];
    if (t != kTet && t != kPrism && t != kHex)
      throw OracleError(E_MESH, "unsupported element at cell " + std::to_string(i));
    m.type[i] = t;
    for (int k = 0; k < t; ++k) {
      int64_t nd = in.cell_nodes[(int64_t)i * 8 + k];
      if (nd < 0 || nd >= in.n_nodes) throw OracleError(E_MESH, "bad node id in cell " + std::to_string(i));
      m.cell_xyz[i].push_back({in.xyz[nd * 3], in.xyz[nd * 3 + 1], in.xyz[nd * 3 + 2]});
    }
  }
  m.geom.resize(m.n_cells);
  for (int i = 0; i < m.n_cells; ++i) {
    m.geom[i] = cell_geometry(m.type[i], m.cell_xyz[i]);
    if (!(m.geom[i].V > 0)) throw OracleError(E_MESH, "degenerate cell " + std::to_string(i));
  }
  // --- faces by sorted node key (std::map) ---
  struct Half { int cell, p; };
  std::map<std::vector<int64_t>, std::vector<Half>> by_key;
  for (int i = 0; i < m.n_cells; ++i)
    for (int p = 0; p < n_faces_of(m.type[i]); ++p) {
      std::vector<int64_t> key;
      for (int ln : face_local_nodes(m.type[i], p)) key.push_back(in.cell_nodes[(int64_t)i * 8 + ln]);
      std::sort(key.begin(), key.end());
      by_key[key].push_back({i, p});
    }
  std::map<std::vector<int64_t>, int> bc_of;
  for (int64_t b = 0; b < in.n_bf; ++b) {
    std::vector<int64_t> key;
    for (int k = 0; k < 4; ++k)
      if (in.bface_nodes[b * 4 + k] >= 0) key.push_back(in.bface_nodes[b * 4 + k]);
    std::sort(key.begin(), key.end());
    bc_of[key] = in.bface_tag[b];
  }
  m.cell_face.assign(m.n_cells, std::vector<int>());
  for (int i = 0; i < m.n_cells; ++i) m.cell_face[i].assign(n_faces_of(m.type[i]), -1);

  auto face_points = [&](int cell, int p) {
    std::vector<Vec3> pts;
    for (int ln : face_local_nodes(m.type[cell], p)) pts.push_back(m.cell_xyz[cell][ln]);
    return pts;
  };
  auto make_face = [&](int owner, int po) {
    Face f;
    f.owner = owner;
    f.gp = face_gauss_points(face_points(owner, po));
    // orient out of the owner: flip if the summed normal points towards its centroid
    Vec3 fc{0, 0, 0}, nsum{0, 0, 0};
    auto pts = face_points(owner, po);
    for (auto& x : pts) fc = add(fc, scale(x, 1.0 / pts.size()));
    for (auto& g : f.gp) nsum = add(nsum, scale(g.n, g.wS));
    if (dot(nsum, sub(fc, m.geom[owner].c)) < 0)
      for (auto& g : f.gp) g.n = scale(g.n, -1.0);
    for (auto& g : f.gp) f.area += g.wS;
    return f;
  };

  std::vector<Half> unmatched;
  for (auto& kv : by_key) {
    auto& hs = kv.second;
    if (hs.size() > 2) throw OracleError(E_MESH, "non-manifold face at cell " + std::to_string(hs[0].cell));
    if (hs.size() == 2) {
      Half a = hs[0], b = hs[1];
      if (b.cell < a.cell) std::swap(a, b);
      Face f = make_face(a.cell, a.p);
      f.nb = b.cell;
      int id = (int)m.faces.size();
      m.faces.push_back(f);
      m.cell_face[a.cell][a.p] = id;
      m.cell_face[b.cell][b.p] = id;
    } else {
      auto it = bc_of.find(kv.first);
      if (it != bc_of.end()) {
        Face f = make_face(hs[0].cell, hs[0].p);
        f.bc = it->second;
        int id = (int)m.faces.size();
        m.faces.push_back(f);
        m.cell_face[hs[0].cell][hs[0].p] = id;
      } else {
        unmatched.push_back(hs[0]);
      }
    }
  }
  // --- periodic pairing by translation (R23): canonical vertex coordinates mod L ---
  const double* L = in.per_len;
  const double* O = in.per_origin;
  double Lmax = std::max(std::max(L[0], L[1]), L[2]);
  double tol = 1e-7 * (Lmax > 0 ? Lmax : 1.0);
  std::map<std::vector<int64_t>, std::vector<Half>> by_pkey;
  for (auto& h : unmatched) {
    auto pts = face_points(h.cell, h.p);
    std::vector<int64_t> key;
    std::vector<std::array<int64_t, 3>> q;
    for (auto& x : pts) {
      std::array<int64_t, 3> qi;
      for (int a = 0; a < 3; ++a) {
        double y = x[a] - O[a];
        if (L[a] > 0) {
          y = std::fmod(y, L[a]);
          if (y < 0) y += L[a];
          if (L[a] - y < tol) y = 0.0;
        }
        qi[a] = (int64_t)std::llround(y / tol);
      }
      q.push_back(qi);
    }
    std::sort(q.begin(), q.end());
    for (auto& qi : q) key.insert(key.end(), qi.begin(), qi.end());
    by_pkey[key].push_back(h);
  }
  for (auto& kv : by_pkey) {
    auto& hs = kv.second;
    if (hs.size() != 2) throw OracleError(E_MESH, "unmatched boundary face at cell " + std::to_string(hs[0].cell));
    Half a = hs[0], b = hs[1];
    if (b.cell < a.cell) std::swap(a, b);
    Face f = make_face(a.cell, a.p);
    f.nb = b.cell;
    Vec3 ca{0, 0, 0}, cb{0, 0, 0};
    auto pa = face_points(a.cell, a.p), pb = face_points(b.cell, b.p);
    for (auto& x : pa) ca = add(ca, scale(x, 1.0 / pa.size()));
    for (auto& x : pb) cb = add(cb, scale(x, 1.0 / pb.size()));
    Vec3 s = sub(ca, cb);
    for (int ax = 0; ax < 3; ++ax) s[ax] = (L[ax] > 0) ? L[ax] * std::round(s[ax] / L[ax]) : 0.0;
    f.shift = s;
    int id = (int)m.faces.size();
    m.faces.push_back(f);
    m.cell_face[a.cell][a.p] = id;
    m.cell_face[b.cell][b.p] = id;
  }
  // --- ghosts for physical boundary faces (Alg. 1 "Add ghost cell according to
  //     boundary condition"; R25: centroid and M2 mirrored across the face) ---
  for (int fi = 0; fi < (int)m.faces.size(); ++fi) {
    Face& f = m.faces[fi];
    if (f.nb >= 0) continue;
    f.ghost = m.n_ghosts++;
    m.ghost_cell.push_back(f.owner);
    m.ghost_face.push_back(fi);
    m.ghost_bc.push_back(f.bc);
    Vec3 xf{0, 0, 0}, nf{0, 0, 0};
    for (auto& g : f.gp) { xf = add(xf, scale(g.x, g.wS / f.area)); nf = add(nf, scale(g.n, g.wS)); }
    nf = scale(nf, 1.0 / norm(nf));
    const CellGeom& gi = m.geom[f.owner];
    CellGeom gg;
    gg.V = gi.V;
    gg.c = sub(gi.c, scale(nf, 2.0 * dot(sub(gi.c, xf), nf)));
    double R[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) R[a][b] = (a == b ? 1.0 : 0.0) - 2.0 * nf[a] * nf[b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int c = 0; c < 3; ++c)
          for (int d = 0; d < 3; ++d) s += R[a][c] * gi.M2[c][d] * R[b][d];
        gg.M2[a][b] = s;
      }
    m.geom.push_back(gg);
  }
  // --- CellNeighbor (one entry per local face) ---
  m.neighbor.assign(m.n_cells, {});
  m.h_dt.assign(m.n_cells, 0.0);
  for (int i = 0; i < m.n_cells; ++i) {
    double smax = 0;
    for (int p = 0; p < (int)m.cell_face[i].size(); ++p) {
      int fi = m.cell_face[i][p];
      if (fi < 0) throw OracleError(E_MESH, "open face at cell " + std::to_string(i));
      const Face& f = m.faces[fi];
      smax = std::max(smax, f.area);
      if (f.nb < 0) m.neighbor[i].push_back({m.n_cells + f.ghost, {0, 0, 0}});
      else if (f.owner == i && f.nb == i) throw OracleError(E_MESH, "self-periodic face");
      else if (f.owner == i) m.neighbor[i].push_back({f.nb, f.shift});
      else m.neighbor[i].push_back({f.owner, scale(f.shift, -1.0)});
    }
    m.h_dt[i] = m.geom[i].V / smax;
  }
  // --- Alg. 1 two-layer big stencil; first layer = ORIGINAL face neighbours (R18) ---
  auto same = [](const Vec3& a, const Vec3& b) {
    return std::fabs(a[0] - b[0]) + std::fabs(a[1] - b[1]) + std::fabs(a[2] - b[2]) < 1e-9;
  };
  m.big.assign(m.n_cells, {});
  m.subs.assign(m.n_cells, {});
  for (int i = 0; i < m.n_cells; ++i) {
    std::vector<Member>& S = m.big[i];
    auto find = [&](int id) -> int {
      for (size_t k = 0; k < S.size(); ++k)
        if (S[k].id == id) return (int)k;
      return -1;
    };
    auto push = [&](const Member& mb) {
      if (mb.id == i) {
        if (!same(mb.s, {0, 0, 0})) throw OracleError(E_MESH, "periodic box too small for the 2-layer stencil");
        return;
      }
      int k = find(mb.id);
      if (k >= 0) {
        if (!same(S[k].s, mb.s)) throw OracleError(E_MESH, "periodic box too small for the 2-layer stencil");
        return;
      }
      S.push_back(mb);
    };
    for (auto& nb : m.neighbor[i]) push(nb);
    for (auto& nb : m.neighbor[i]) {
      if (nb.id >= m.n_cells) continue;  // a ghost has no neighbours of its own
      for (auto& nn : m.neighbor[nb.id]) {
        if (nn.id >= m.n_cells) {
          // second-layer ghost: reflected about its own face; only meaningful
          // with zero periodic shift (physical boundaries are not periodic)
          push({nn.id, nb.s});
        } else {
          push({nn.id, add(nb.s, nn.s)});
        }
      }
    }
    // sub-stencils
    const auto& F = m.neighbor[i];
    if (m.type[i] == kTet) {
      // R16: triples {1,2,3},{1,2,4},{2,3,4},{3,1,4} with neighbours of i_1..i_4
      const int tri[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {2, 0, 3}};
      for (int mm = 0; mm < 4; ++mm) {
        std::vector<Member> Sm;
        auto pushm = [&](const Member& mb) {
          if (mb.id == i) return;
          for (auto& e : Sm)
            if (e.id == mb.id) return;
          Sm.push_back(mb);
        };
        for (int k = 0; k < 3; ++k) pushm(F[tri[mm][k]]);
        const Member& im = F[mm];
        if (im.id < m.n_cells)
          for (auto& nn : m.neighbor[im.id]) {
            if (nn.id >= m.n_cells) pushm({nn.id, im.s});
            else pushm({nn.id, add(im.s, nn.s)});
          }
        m.subs[i].push_back(Sm);
      }
    } else if (m.type[i] == kPrism) {
      // R30 (the paper gives no prism rule; the hex pattern of P:390-395 transferred): one
      // triangle neighbour (face 0 or 1) with two ring-adjacent side neighbours, 2 x 3 = 6
      const int ps[6][3] = {{0, 2, 3}, {0, 3, 4}, {0, 4, 2}, {1, 2, 3}, {1, 3, 4}, {1, 4, 2}};
      for (int mm = 0; mm < 6; ++mm) {
        std::vector<Member> Sm;
        for (int k = 0; k < 3; ++k) Sm.push_back(F[ps[mm][k]]);
        m.subs[i].push_back(Sm);
      }
    } else {
      // P:390-395 with faces 0/5 opposed and ring 1..4
      const int hs[8][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 4}, {0, 4, 1}, {5, 1, 2}, {5, 2, 3}, {5, 3, 4}, {5, 4, 1}};
      for (int mm = 0; mm < 8; ++mm) {
        std::vector<Member> Sm;
        for (int k = 0; k < 3; ++k) Sm.push_back(F[hs[mm][k]]);
        m.subs[i].push_back(Sm);
      }
    }
  }
  return m;
}

// ---------------------------------------------------------------------------
// O4 Least squares (R20): Householder QR of the scaled, centred system
// ---------------------------------------------------------------------------
// Solves min ||A x - B||_2 column by column; A is m x n (m >= n), row-major.
bool householder_lsq(int mrows, int ncols, std::vector<double> A, std::vector<double>& B, int nrhs,
                     std::vector<double>& X) {
  std::vector<double> diag(ncols);
  double amax = 0;
  for (double v : A) amax = std::max(amax, std::fabs(v));
  for (int k = 0; k < ncols; ++k) {
    double nrm = 0;
    for (int r = k; r < mrows; ++r) nrm += A[r * ncols + k] * A[r * ncols + k];
    nrm = std::sqrt(nrm);
    if (nrm <= 1e-12 * amax) return false;
    double alpha = A[k * ncols + k] > 0 ? -nrm : nrm;
    std::vector<double> v(mrows, 0.0);
    for (int r = k; r < mrows; ++r) v[r] = A[r * ncols + k];
    v[k] -= alpha;
    double vv = 0;
    for (int r = k; r < mrows; ++r) vv += v[r] * v[r];
    if (vv > 0) {
      for (int c = k; c < ncols; ++c) {
        double s = 0;
        for (int r = k; r < mrows; ++r) s += v[r] * A[r * ncols + c];
        s = 2.0 * s / vv;
        for (int r = k; r < mrows; ++r) A[r * ncols + c] -= s * v[r];
      }
      for (int c = 0; c < nrhs; ++c) {
        double s = 0;
        for (int r = k; r < mrows; ++r) s += v[r] * B[r * nrhs + c];
        s = 2.0 * s / vv;
        for (int r = k; r < mrows; ++r) B[r * nrhs + c] -= s * v[r];
      }
    }
    diag[k] = A[k * ncols + k];
  }
  X.assign(ncols * nrhs, 0.0);
  for (int c = 0; c < nrhs; ++c)
    for (int k = ncols - 1; k >= 0; --k) {
      double s = B[k * nrhs + c];
      for (int j = k + 1; j < ncols; ++j) s -= A[k * ncols + j] * X[j * nrhs + c];
      X[k * nrhs + c] = s / A[k * ncols + k];
    }
  return true;
}

// Cell polynomials of one cell (Eq. polys), coefficients of the
// basis p_d(x) = (x-c_i)^d - mean_{Omega_i}(x-c_i)^d in physical units.
// d order: x, y, z, xx, yy, zz, xy, xz, yz.
struct CellPolys {
  double a[9][5];                // P_0 (quadratic), per conserved variable
  std::vector<std::array<std::array<double, 5>, 3>> b;  // P_m (linear), m = 1..M
  std::vector<std::array<double, 5>> wbar;               // omega-bar_0..M per variable
  double Q[5];
  std::vector<std::array<double, 5>> beta;               // beta_0..M
};

const int kQuadIdx[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};

struct State {
  const Mesh* mesh;
  const double* Q;          // [n_cells][5]
  std::vector<double> Qg;   // ghost states [n_ghosts][5]
  const double* cell_Q(int id) const {
    return id < mesh->n_cells ? Q + (size_t)id * 5 : Qg.data() + (size_t)(id - mesh->n_cells) * 5;
  }
};

// fit P_0 over the big stencil and P_m over each sub-stencil by least squares
CellPolys fit_cell(const Mesh& m, const State& st, int i, const Config& cfg) {
  CellPolys P;
  const CellGeom& gi = m.geom[i];
  const double h = std::cbrt(gi.V);
  const double* Qi = st.cell_Q(i);
  for (int v = 0; v < 5; ++v) P.Q[v] = Qi[v];
  auto row = [&](const Member& mb, double* r9) {
    const CellGeom& gk = m.geom[mb.id];
    Vec3 D = sub(add(gk.c, mb.s), gi.c);  // centroid offset of the member image
    for (int a = 0; a < 3; ++a) r9[a] = D[a] / h;
    for (int q = 0; q < 6; ++q) {
      int a = kQuadIdx[q][0], b = kQuadIdx[q][1];
      // mean over Omega_k of (x-c_i)_a (x-c_i)_b minus mean over Omega_i (zero-mean basis)
      r9[3 + q] = (gk.M2[a][b] + D[a] * D[b] - gi.M2[a][b]) / (h * h);
    }
  };
  // P_0: rows = big-stencil cells other than i
  {
    const auto& S = m.big[i];
    int mr = (int)S.size();
    std::vector<double> A(mr * 9), B(mr * 5), X;
    for (int k = 0; k < mr; ++k) {
      row(S[k], &A[k * 9]);
      const double* Qk = st.cell_Q(S[k].id);
      for (int v = 0; v < 5; ++v) B[k * 5 + v] = Qk[v] - Qi[v];
    }
    if (mr < 9 || !householder_lsq(mr, 9, A, B, 5, X))
      throw OracleError(E_STENCIL, "rank-deficient big stencil at cell " + std::to_string(i));
    for (int d = 0; d < 9; ++d)
      for (int v = 0; v < 5; ++v) P.a[d][v] = X[d * 5 + v] / (d < 3 ? h : h * h);
  }
  for (const auto& Sm : m.subs[i]) {
    int mr = (int)Sm.size();
    std::vector<double> A(mr * 3), B(mr * 5), X;
    for (int k = 0; k < mr; ++k) {
      double r9[9];
      row(Sm[k], r9);
      for (int a = 0; a < 3; ++a) A[k * 3 + a] = r9[a];
      const double* Qk = st.cell_Q(Sm[k].id);
      for (int v = 0; v < 5; ++v) B[k * 5 + v] = Qk[v] - Qi[v];
    }
    if (mr < 3 || !householder_lsq(mr, 3, A, B, 5, X))
      throw OracleError(E_STENCIL, "rank-deficient sub-stencil at cell " + std::to_string(i));
    std::array<std::array<double, 5>, 3> b;
    for (int d = 0; d < 3; ++d)
      for (int v = 0; v < 5; ++v) b[d][v] = X[d * 5 + v] / h;
    P.b.push_back(b);
  }
  // --- smoothness indicators by exact quadrature over Omega_i ---
  const int M = (int)P.b.size();
  std::vector<Vec3> pts;
  std::vector<double> wts;
  if (i < m.n_cells) cell_quadrature(m.type[i], m.cell_xyz[i], pts, wts);
  const double V = gi.V;
  P.beta.assign(M + 1, {});
  for (int v = 0; v < 5; ++v) {
    // beta_0: |l| = 1 terms V^{-1/3} int (d_a P0)^2, |l| = 2 terms V^{1/3} int (d^l P0)^2
    double s1 = 0;
    for (size_t q = 0; q < pts.size(); ++q) {
      Vec3 X = sub(pts[q], gi.c);
      double gx = P.a[0][v] + 2 * P.a[3][v] * X[0] + P.a[6][v] * X[1] + P.a[7][v] * X[2];
      double gy = P.a[1][v] + 2 * P.a[4][v] * X[1] + P.a[6][v] * X[0] + P.a[8][v] * X[2];
      double gz = P.a[2][v] + 2 * P.a[5][v] * X[2] + P.a[7][v] * X[0] + P.a[8][v] * X[1];
      s1 += wts[q] * (gx * gx + gy * gy + gz * gz);
    }
    // second derivatives are constant: d_xx P = 2 a_xx, d_xy P = a_xy, ... (each
    // multi-index l counted once, R15); int over Omega_i = V * value^2
    double dxx = 2 * P.a[3][v], dyy = 2 * P.a[4][v], dzz = 2 * P.a[5][v];
    double dxy = P.a[6][v], dxz = P.a[7][v], dyz = P.a[8][v];
    double s2 = V * (dxx * dxx + dyy * dyy + dzz * dzz + dxy * dxy + dxz * dxz + dyz * dyz);
    P.beta[0][v] = std::pow(V, -1.0 / 3.0) * s1 + std::pow(V, 1.0 / 3.0) * s2;
    for (int mm = 0; mm < M; ++mm) {
      double bx = P.b[mm][0][v], by = P.b[mm][1][v], bz = P.b[mm][2][v];
      P.beta[mm + 1][v] = std::pow(V, -1.0 / 3.0) * (V * (bx * bx + by * by + bz * bz));
    }
  }
  // --- nonlinear weights ---
  const double gm = 0.025, g0 = 1.0 - gm * M;
  P.wbar.assign(M + 1, {});
  for (int v = 0; v < 5; ++v) {
    double tauZ = 0;
    for (int mm = 1; mm <= M; ++mm) tauZ += std::fabs(P.beta[0][v] - P.beta[mm][v]) / M;
    std::vector<double> w(M + 1);
    double sum = 0;
    for (int mm = 0; mm <= M; ++mm) {
      double gam = mm == 0 ? g0 : gm;
      double r = tauZ / (P.beta[mm][v] + cfg.eps);
      w[mm] = gam * (1.0 + (cfg.omega_pow == 2 ? r * r : r));
      sum += w[mm];
    }
    for (int mm = 0; mm <= M; ++mm) P.wbar[mm][v] = w[mm] / sum;
  }
  (void)cfg;
  return P;
}

// Eq. (weno), evaluated literally at point x (cell i's coordinates):
// value and gradient per conserved variable.  linear = true replaces the normalized
// nonlinear weights omega-bar_m by the linear weights gamma_m (SPEC's central-gradient
// recombination, reading R9s).
void weno_point(const Mesh& m, const CellPolys& P, int i, const Vec3& x, double val[5], double grad[5][3],
                bool linear = false) {
  const CellGeom& gi = m.geom[i];
  Vec3 X = sub(x, gi.c);
  const int M = (int)P.b.size();
  const double gm = 0.025, g0 = 1.0 - gm * M;
  double mono[9] = {X[0], X[1], X[2], X[0] * X[0] - gi.M2[0][0], X[1] * X[1] - gi.M2[1][1], X[2] * X[2] - gi.M2[2][2],
                    X[0] * X[1] - gi.M2[0][1], X[0] * X[2] - gi.M2[0][2], X[1] * X[2] - gi.M2[1][2]};
  for (int v = 0; v < 5; ++v) {
    // P_0 and its gradient
    double p0 = P.Q[v];
    for (int d = 0; d < 9; ++d) p0 += P.a[d][v] * mono[d];
    double g0v[3] = {P.a[0][v] + 2 * P.a[3][v] * X[0] + P.a[6][v] * X[1] + P.a[7][v] * X[2],
                     P.a[1][v] + 2 * P.a[4][v] * X[1] + P.a[6][v] * X[0] + P.a[8][v] * X[2],
                     P.a[2][v] + 2 * P.a[5][v] * X[2] + P.a[7][v] * X[0] + P.a[8][v] * X[1]};
    double sum_gP = 0, sum_wP = 0, sum_gG[3] = {0, 0, 0}, sum_wG[3] = {0, 0, 0};
    for (int mm = 0; mm < M; ++mm) {
      const double wb = linear ? gm : P.wbar[mm + 1][v];
      double pm = P.Q[v] + P.b[mm][0][v] * X[0] + P.b[mm][1][v] * X[1] + P.b[mm][2][v] * X[2];
      sum_gP += gm / g0 * pm;
      sum_wP += wb * pm;
      for (int a = 0; a < 3; ++a) {
        sum_gG[a] += gm / g0 * P.b[mm][a][v];
        sum_wG[a] += wb * P.b[mm][a][v];
      }
    }
    const double wb0 = linear ? g0 : P.wbar[0][v];
    val[v] = wb0 * (p0 / g0 - sum_gP) + sum_wP;
    for (int a = 0; a < 3; ++a) grad[v][a] = wb0 * (g0v[a] / g0 - sum_gG[a]) + sum_wG[a];
  }
}

// ---------------------------------------------------------------------------
// Kinetic part: Maxwellian moments, slopes, Eq. (flux)
// ---------------------------------------------------------------------------
struct Maxw {
  double rho, U, V, W, lam;
};

Maxw maxwellian_of(const double q[5], double K) {
  Maxw g;
  g.rho = q[0];
  g.U = q[1] / q[0];
  g.V = q[2] / q[0];
  g.W = q[3] / q[0];
  // rhoE = 1/2 rho |U|^2 + (K+3) rho / (4 lambda)
  g.lam = (K + 3.0) * g.rho / (4.0 * (q[4] - 0.5 * g.rho * (g.U * g.U + g.V * g.V + g.W * g.W)));
  return g;
}

enum Range { kFull, kPos, kNeg };

// <u^a>, <v^b>, <w^c>, <xi^{2d}> of g/rho; the u-moments over the full line or
// the half lines u > 0 / u < 0.
struct Moments {
  double u[8], v[8], w[8], xi[3];
};

Moments moments_of(const Maxw& g, Range r, double K) {
  Moments M;
  const double PI = 3.14159265358979323846;
  double sl = std::sqrt(g.lam);
  if (r == kFull) {
    M.u[0] = 1.0;
    M.u[1] = g.U;
  } else {
    double e = std::exp(-g.lam * g.U * g.U);
    if (r == kPos) {
      M.u[0] = 0.5 * std::erfc(-sl * g.U);
      M.u[1] = g.U * M.u[0] + 0.5 * e / std::sqrt(PI * g.lam);
    } else {
      M.u[0] = 0.5 * std::erfc(sl * g.U);
      M.u[1] = g.U * M.u[0] - 0.5 * e / std::sqrt(PI * g.lam);
    }
  }
  M.v[0] = 1.0; M.v[1] = g.V;
  M.w[0] = 1.0; M.w[1] = g.W;
  for (int n = 0; n + 2 < 8; ++n) {
    M.u[n + 2] = g.U * M.u[n + 1] + (n + 1) / (2.0 * g.lam) * M.u[n];
    M.v[n + 2] = g.V * M.v[n + 1] + (n + 1) / (2.0 * g.lam) * M.v[n];
    M.w[n + 2] = g.W * M.w[n + 1] + (n + 1) / (2.0 * g.lam) * M.w[n];
  }
  M.xi[0] = 1.0;
  M.xi[1] = K / (2.0 * g.lam);
  M.xi[2] = K * (K + 2.0) / (4.0 * g.lam * g.lam);
  return M;
}

// Polynomials in (u, v, w, xi^2): sum of c * u^a v^b w^c (xi^2)^d
struct Term {
  double c;
  int a, b, cc, d;
};
using Poly = std::vector<Term>;

Poly make_psi(int i) {  // collision invariants psi = (1, u, v, w, 1/2(u^2+v^2+w^2+xi^2))
  switch (i) {
    case 0: return {{1.0, 0, 0, 0, 0}};
    case 1: return {{1.0, 1, 0, 0, 0}};
    case 2: return {{1.0, 0, 1, 0, 0}};
    case 3: return {{1.0, 0, 0, 1, 0}};
    default: return {{0.5, 2, 0, 0, 0}, {0.5, 0, 2, 0, 0}, {0.5, 0, 0, 2, 0}, {0.5, 0, 0, 0, 1}};
  }
}
const Poly& psi(int i) {
  static const Poly P[5] = {make_psi(0), make_psi(1), make_psi(2), make_psi(3), make_psi(4)};
  return P[i];
}
Poly mul(const Poly& p, const Poly& q) {
  Poly r;
  for (auto& s : p)
    for (auto& t : q) r.push_back({s.c * t.c, s.a + t.a, s.b + t.b, s.cc + t.cc, s.d + t.d});
  return r;
}
Poly addp(const Poly& p, const Poly& q) {
  Poly r = p;
  r.insert(r.end(), q.begin(), q.end());
  return r;
}
Poly slope_poly(const double a[5]) {  // a = a_1 + a_2 u + a_3 v + a_4 w + a_5 psi_5
  Poly r;
  for (int j = 0; j < 5; ++j)
    for (auto t : psi(j)) {
      t.c *= a[j];
      r.push_back(t);
    }
  return r;
}
const Poly kU = {{1.0, 1, 0, 0, 0}}, kV = {{1.0, 0, 1, 0, 0}}, kW = {{1.0, 0, 0, 1, 0}};

// <p> = sum over terms of c <u^a><v^b><w^c><xi^2d> (moments factorise)
double moment(const Poly& p, const Moments& M) {
  double s = 0;
  for (auto& t : p) s += t.c * M.u[t.a] * M.v[t.b] * M.w[t.cc] * M.xi[t.d];
  return s;
}
// <p q> and <p q r> without forming the product polynomial
double moment2(const Poly& p, const Poly& q, const Moments& M) {
  double s = 0;
  for (auto& x : p)
    for (auto& y : q) s += x.c * y.c * M.u[x.a + y.a] * M.v[x.b + y.b] * M.w[x.cc + y.cc] * M.xi[x.d + y.d];
  return s;
}
double moment3(const Poly& p, const Poly& q, const Poly& r, const Moments& M) {
  double s = 0;
  for (auto& x : p)
    for (auto& y : q)
      for (auto& z : r)
        s += x.c * y.c * z.c * M.u[x.a + y.a + z.a] * M.v[x.b + y.b + z.b] * M.w[x.cc + y.cc + z.cc] *
             M.xi[x.d + y.d + z.d];
  return s;
}

// Gaussian elimination with partial pivoting (5x5)
void solve5(double A[5][5], double b[5], double x[5]) {
  double M[5][6];
  for (int i = 0; i < 5; ++i) {
    for (int j = 0; j < 5; ++j) M[i][j] = A[i][j];
    M[i][5] = b[i];
  }
  for (int k = 0; k < 5; ++k) {
    int piv = k;
    for (int r = k + 1; r < 5; ++r)
      if (std::fabs(M[r][k]) > std::fabs(M[piv][k])) piv = r;
    for (int j = 0; j < 6; ++j) std::swap(M[k][j], M[piv][j]);
    for (int r = k + 1; r < 5; ++r) {
      double f = M[r][k] / M[k][k];
      for (int j = k; j < 6; ++j) M[r][j] -= f * M[k][j];
    }
  }
  for (int k = 4; k >= 0; --k) {
    double s = M[k][5];
    for (int j = k + 1; j < 5; ++j) s -= M[k][j] * x[j];
    x[k] = s / M[k][k];
  }
}

// micro-slope a with <a> = rho <a psi> = b, i.e. sum_j a_j <psi_i psi_j> = b_i / rho
void micro_slope(const Moments& F, double rho, const double b[5], double a[5]) {
  double A[5][5], rhs[5];
  for (int i = 0; i < 5; ++i) {
    for (int j = 0; j < 5; ++j) A[i][j] = moment2(psi(i), psi(j), F);
    rhs[i] = b[i] / rho;
  }
  solve5(A, rhs, a);
}

// Spatial slopes a_1, a_2, a_3 (local n, t1, t2) from derivatives, and the
// temporal slope A from compatibility <a_1 u + a_2 v + a_3 w + A> = 0.
struct Slopes {
  double a[3][5];
  double A[5];
};

Slopes slopes_of(const Maxw& g, const Moments& F, const double dq[3][5]) {
  Slopes s;
  for (int j = 0; j < 3; ++j) micro_slope(F, g.rho, dq[j], s.a[j]);
  Poly au = addp(addp(mul(slope_poly(s.a[0]), kU), mul(slope_poly(s.a[1]), kV)), mul(slope_poly(s.a[2]), kW));
  double b[5];
  for (int i = 0; i < 5; ++i) b[i] = -g.rho * moment2(au, psi(i), F);
  micro_slope(F, g.rho, b, s.A);
  return s;
}

// moment vectors of one Maxwellian: <u psi>, <(a.u) u psi>, <A u psi> (normalised by rho)
void flux_moments(const Slopes& s, const Moments& M, double m1[5], double m2[5], double m3[5]) {
  Poly au = addp(addp(mul(slope_poly(s.a[0]), kU), mul(slope_poly(s.a[1]), kV)), mul(slope_poly(s.a[2]), kW));
  Poly Ap = slope_poly(s.A);
  for (int i = 0; i < 5; ++i) {
    m1[i] = moment2(kU, psi(i), M);
    m2[i] = moment3(au, kU, psi(i), M);
    m3[i] = moment3(Ap, kU, psi(i), M);
  }
}

struct GpFluxOut {
  double I_half[5], I_full[5];  // time integrals over [0, dt/2] and [0, dt] (local frame)
  double F[5], dF[5];           // fitted F^n and d_t F^n (local frame)
  double Q0[5];
  double dq0[3][5];             // equilibrium slopes dQ0 used (local frame), per dq0_mode
  double tau;
};

// One Gauss point, local frame (x = normal): left state (value + derivatives
// along n, t1, t2), right state, step dt.  Eq. (flux).  dq0_ext: the
// equilibrium slopes dQ0 when they come from outside (dq0_mode 2), else NULL.
GpFluxOut gks_flux_local(const double ql[5], const double dql[3][5], const double qr[5], const double dqr[3][5],
                         double dt, const Config& cfg, const double (*dq0_ext)[5] = nullptr) {
  const double K = cfg.K();
  GpFluxOut out;
  Maxw gl = maxwellian_of(ql, K), gr = maxwellian_of(qr, K);
  Moments Ml_pos = moments_of(gl, kPos, K), Ml_full = moments_of(gl, kFull, K);
  Moments Mr_neg = moments_of(gr, kNeg, K), Mr_full = moments_of(gr, kFull, K);
  // Q0 by compatibility: int_{u>0} psi g_l + int_{u<0} psi g_r
  double Q0[5];
  for (int i = 0; i < 5; ++i) Q0[i] = gl.rho * moment(psi(i), Ml_pos) + gr.rho * moment(psi(i), Mr_neg);
  Maxw g0 = maxwellian_of(Q0, K);
  Moments M0 = moments_of(g0, kFull, K);
  // slopes: l, r from their derivatives (<a^k_j> = dQ_k/dn_j)
  Slopes sl = slopes_of(gl, Ml_full, dql);
  Slopes sr = slopes_of(gr, Mr_full, dqr);
  // equilibrium slopes from dQ0 (<a-bar_j> = dQ0/dn_j; how dQ0 is obtained is
  // not printed):
  double dq0[3][5];
  for (int j = 0; j < 3; ++j)
    for (int v = 0; v < 5; ++v) {
      if (cfg.dq0_mode == 0) {
        dq0[j][v] = 0.5 * (dql[j][v] + dqr[j][v]);  // R9: average of the two gradients
      } else if (cfg.dq0_mode == 1) {
        // R9k: the j-derivative of the compatibility definition Q0 = int_{u>0} psi g_l +
        // int_{u<0} psi g_r with d_j g_k = a^k_j g_k
        dq0[j][v] = gl.rho * moment2(slope_poly(sl.a[j]), psi(v), Ml_pos) +
                    gr.rho * moment2(slope_poly(sr.a[j]), psi(v), Mr_neg);
      } else {
        if (!dq0_ext) throw OracleError(E_ARG, "dq0_mode 2 needs the linear-weight gradients");
        dq0[j][v] = dq0_ext[j][v];  // R9s: computed by the caller from the gamma-weighted polynomials
      }
    }
  Slopes s0 = slopes_of(g0, M0, dq0);
  for (int j = 0; j < 3; ++j)
    for (int v = 0; v < 5; ++v) out.dq0[j][v] = dq0[j][v];
  // collision time (R7)
  double tau = 0.0;
  if (cfg.tau_mode == 1) {
    double p0 = g0.rho / (2.0 * g0.lam), pl = gl.rho / (2.0 * gl.lam), pr = gr.rho / (2.0 * gr.lam);
    double T0 = p0 / g0.rho;
    double mu = cfg.mu_inf * std::pow(T0 / cfg.t_inf, cfg.mu_exp);
    tau = mu / p0 + cfg.c1 * std::fabs(pl - pr) / (pl + pr) * dt;
  }
  out.tau = tau;
  double e0[5], e1[5], e2[5], l1[5], l2[5], l3[5], r1[5], r2[5], r3[5];
  flux_moments(s0, M0, e0, e1, e2);
  flux_moments(sl, Ml_pos, l1, l2, l3);
  flux_moments(sr, Mr_neg, r1, r2, r3);
  auto integral = [&](double delta, double I[5]) {
    // closed-form time integrals of the five coefficients of Eq. (flux) over [0, delta]
    double e = std::exp(-delta / tau);
    double c1 = delta - tau * (1 - e);
    double c2 = 2 * tau * tau * (1 - e) - tau * delta * (1 + e);
    double c3 = delta * delta / 2 - tau * delta + tau * tau * (1 - e);
    double c4 = tau * (1 - e);
    double c5 = -2 * tau * tau * (1 - e) + tau * delta * e;
    double c6 = -tau * tau * (1 - e);
    for (int i = 0; i < 5; ++i)
      I[i] = g0.rho * (c1 * e0[i] + c2 * e1[i] + c3 * e2[i]) + gl.rho * (c4 * l1[i] + c5 * l2[i] + c6 * l3[i]) +
             gr.rho * (c4 * r1[i] + c5 * r2[i] + c6 * r3[i]);
  };
  integral(0.5 * dt, out.I_half);
  integral(dt, out.I_full);
  // Prandtl-number correction (R29; Xu's heat-flux fix, P:1203-1210 runs a viscous sphere but
  // prints no Pr): the energy flux gains (1/Pr - 1) times the time integral of the heat flux
  // q(t) = 1/2 int (u - U0)((u - U0)^2 + (v - V0)^2 + (w - W0)^2 + xi^2) f_neq dXi, U0 the
  // velocity of Q0, of the non-equilibrium part f_neq = f - g0 (1 + A-bar t) of Eq. (flux)
  // (zero at tau = 0; the Chapman-Enskog heat flux in the Navier-Stokes limit).
  if (cfg.prandtl != 1.0) {
    const Poly cu = {{1.0, 1, 0, 0, 0}, {-g0.U, 0, 0, 0, 0}}, cv = {{1.0, 0, 1, 0, 0}, {-g0.V, 0, 0, 0, 0}},
               cw = {{1.0, 0, 0, 1, 0}, {-g0.W, 0, 0, 0, 0}};
    Poly sq = addp(addp(addp(mul(cu, cu), mul(cv, cv)), mul(cw, cw)), Poly{{1.0, 0, 0, 0, 1}});
    Poly qp = mul(Poly{{0.5, 0, 0, 0, 0}}, mul(cu, sq));
    auto au_of = [](const Slopes& sk) {
      return addp(addp(mul(slope_poly(sk.a[0]), kU), mul(slope_poly(sk.a[1]), kV)), mul(slope_poly(sk.a[2]), kW));
    };
    // heat-flux moments of each term of f_neq (rho-weighted)
    const double q0a = g0.rho * moment2(qp, au_of(s0), M0), q0A = g0.rho * moment2(qp, slope_poly(s0.A), M0);
    const double ql1 = gl.rho * moment(qp, Ml_pos), qla = gl.rho * moment2(qp, au_of(sl), Ml_pos),
                 qlA = gl.rho * moment2(qp, slope_poly(sl.A), Ml_pos);
    const double qr1 = gr.rho * moment(qp, Mr_neg), qra = gr.rho * moment2(qp, au_of(sr), Mr_neg),
                 qrA = gr.rho * moment2(qp, slope_poly(sr.A), Mr_neg);
    auto qint = [&](double delta) {
      double e = std::exp(-delta / tau);
      double c2 = 2 * tau * tau * (1 - e) - tau * delta * (1 + e);
      double c3n = tau * tau * (1 - e) - tau * delta;  // A-bar g0 coefficient of f_neq: tau (e^{-t/tau} - 1)
      double c4 = tau * (1 - e);
      double c5 = -2 * tau * tau * (1 - e) + tau * delta * e;
      double c6 = -tau * tau * (1 - e);
      return c2 * q0a + c3n * q0A + c4 * (ql1 + qr1) + c5 * (qla + qra) + c6 * (qlA + qrA);
    };
    const double fac = 1.0 / cfg.prandtl - 1.0;
    out.I_half[4] += fac * qint(0.5 * dt);
    out.I_full[4] += fac * qint(dt);
  }
  // 2x2 fit: F dt + 1/2 dF dt^2 = I_full ; 1/2 F dt + 1/8 dF dt^2 = I_half
  for (int i = 0; i < 5; ++i) {
    out.F[i] = (4.0 * out.I_half[i] - out.I_full[i]) / dt;
    out.dF[i] = 4.0 * (out.I_full[i] - 2.0 * out.I_half[i]) / (dt * dt);
    out.Q0[i] = Q0[i];
  }
  return out;
}

// Local frame (R11): t1 = normalize(n x e*), e* the axis with smallest |n.e|; t2 = n x t1
void local_frame(const Vec3& n, Vec3& t1, Vec3& t2) {
  int k = 0;
  for (int a = 1; a < 3; ++a)
    if (std::fabs(n[a]) < std::fabs(n[k])) k = a;
  Vec3 e{0, 0, 0};
  e[k] = 1.0;
  t1 = cross(n, e);
  t1 = scale(t1, 1.0 / norm(t1));
  t2 = cross(n, t1);
}

double pressure_of(const double q[5], double gamma) {
  return (gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
}

// ---------------------------------------------------------------------------
// Boundary states (R25): wall mirror and farfield Riemann invariants
// ---------------------------------------------------------------------------
void farfield_state(const double qi[5], const Vec3& n, const Config& cfg, double qb[5]) {
  const double g = cfg.gamma;
  double rho_i = qi[0];
  Vec3 ui{qi[1] / rho_i, qi[2] / rho_i, qi[3] / rho_i};
  double p_i = pressure_of(qi, g);
  double c_i = std::sqrt(g * p_i / rho_i);
  double rho_f = cfg.fs[0], p_f = cfg.fs[4];
  Vec3 uf{cfg.fs[1], cfg.fs[2], cfg.fs[3]};
  double c_f = std::sqrt(g * p_f / rho_f);
  double un_i = dot(ui, n), un_f = dot(uf, n);
  double Rp = un_i + 2 * c_i / (g - 1), Rm = un_f - 2 * c_f / (g - 1);
  if (un_f + c_f < 0) Rp = un_f + 2 * c_f / (g - 1);  // supersonic inflow: both from free stream
  if (un_i - c_i > 0) Rm = un_i - 2 * c_i / (g - 1);  // supersonic outflow: both from interior
  double un = 0.5 * (Rp + Rm), c = 0.25 * (g - 1) * (Rp - Rm);
  Vec3 ut;
  double s;
  if (un > 0) {  // outflow: tangential velocity and entropy from the interior
    ut = sub(ui, scale(n, un_i));
    s = p_i / std::pow(rho_i, g);
  } else {
    ut = sub(uf, scale(n, un_f));
    s = p_f / std::pow(rho_f, g);
  }
  double rho = std::pow(c * c / (g * s), 1.0 / (g - 1));
  double p = rho * c * c / g;
  Vec3 u = add(ut, scale(n, un));
  qb[0] = rho;
  qb[1] = rho * u[0];
  qb[2] = rho * u[1];
  qb[3] = rho * u[2];
  qb[4] = p / (g - 1) + 0.5 * rho * dot(u, u);
}

// ---------------------------------------------------------------------------
// Solver: O8/O9 (Alg. 2)
// ---------------------------------------------------------------------------
struct Solver {
  Mesh mesh;
  Config cfg;
  std::vector<double> Q;  // [n][5]
  double t = 0.0;
  long long fallbacks = 0;
  int threads = 1;
  double last_dt = 0.0;
};

void ghost_states(const Mesh& m, const Config& cfg, State& st) {
  st.Qg.assign((size_t)m.n_ghosts * 5, 0.0);
  for (int g = 0; g < m.n_ghosts; ++g) {
    const double* qi = st.Q + (size_t)m.ghost_cell[g] * 5;
    double* qg = &st.Qg[(size_t)g * 5];
    if (m.ghost_bc[g] == kWall) {
      qg[0] = qi[0]; qg[1] = -qi[1]; qg[2] = -qi[2]; qg[3] = -qi[3]; qg[4] = qi[4];
    } else {
      const Face& f = m.faces[m.ghost_face[g]];
      Vec3 nf{0, 0, 0};
      for (auto& gp : f.gp) nf = add(nf, scale(gp.n, gp.wS));
      nf = scale(nf, 1.0 / norm(nf));
      farfield_state(qi, nf, cfg, qg);
    }
  }
}

// L(Q) and d_t L(Q) (P:240-244 with the fit of P:341-358) for a state Q and step dt.
void residual(Solver& S, const double* Q, double dt, std::vector<double>& L, std::vector<double>& dL,
              long long* fallback_count) {
  const Mesh& m = S.mesh;
  const Config& cfg = S.cfg;
  State st{&m, Q, {}};
  ghost_states(m, cfg, st);
  std::vector<CellPolys> polys(m.n_cells);
#pragma omp parallel for schedule(dynamic, 64) num_threads(S.threads)
  for (int i = 0; i < m.n_cells; ++i) polys[i] = fit_cell(m, st, i, cfg);
  const int nf = (int)m.faces.size();
  std::vector<std::array<double, 5>> Ff(nf), dFf(nf);
  long long fb = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(S.threads) reduction(+ : fb)
  for (int fi = 0; fi < nf; ++fi) {
    const Face& f = m.faces[fi];
    std::array<double, 5> Fs{}, dFs{};
    for (const GaussPoint& gp : f.gp) {
      // values and gradients of both sides at the Gauss point (global frame)
      double vl[5], gl[5][3], vr[5], gr[5][3];
      bool fell_l = false, fell_r = false;
      weno_point(m, polys[f.owner], f.owner, gp.x, vl, gl);
      if (vl[0] <= 0 || pressure_of(vl, cfg.gamma) <= 0) {  // R21 positivity fallback
        ++fb;
        fell_l = true;
        for (int v = 0; v < 5; ++v) {
          vl[v] = Q[(size_t)f.owner * 5 + v];
          gl[v][0] = gl[v][1] = gl[v][2] = 0;
        }
      }
      Vec3 n = gp.n, t1, t2;
      local_frame(n, t1, t2);
      const Vec3 dir[3] = {n, t1, t2};
      auto to_local = [&](const double val[5], const double grad[5][3], double q[5], double dq[3][5]) {
        q[0] = val[0];
        q[4] = val[4];
        Vec3 mom{val[1], val[2], val[3]};
        q[1] = dot(mom, n); q[2] = dot(mom, t1); q[3] = dot(mom, t2);
        for (int j = 0; j < 3; ++j) {
          // derivative along dir[j] of each variable, momentum rotated
          double d[5];
          for (int v = 0; v < 5; ++v) d[v] = grad[v][0] * dir[j][0] + grad[v][1] * dir[j][1] + grad[v][2] * dir[j][2];
          Vec3 dm{d[1], d[2], d[3]};
          dq[j][0] = d[0];
          dq[j][1] = dot(dm, n); dq[j][2] = dot(dm, t1); dq[j][3] = dot(dm, t2);
          dq[j][4] = d[4];
        }
      };
      double ql[5], dql[3][5], qr[5], dqr[3][5];
      to_local(vl, gl, ql, dql);
      if (f.nb >= 0) {
        weno_point(m, polys[f.nb], f.nb, sub(gp.x, f.shift), vr, gr);
        if (vr[0] <= 0 || pressure_of(vr, cfg.gamma) <= 0) {
          ++fb;
          fell_r = true;
          for (int v = 0; v < 5; ++v) {
            vr[v] = Q[(size_t)f.nb * 5 + v];
            gr[v][0] = gr[v][1] = gr[v][2] = 0;
          }
        }
        to_local(vr, gr, qr, dqr);
      } else if (f.bc == kWall) {
        // mirror (R25): normal velocity and tangential velocities reversed;
        // normal derivatives negated
        for (int v = 0; v < 5; ++v) {
          double sv = (v >= 1 && v <= 3) ? -1.0 : 1.0;
          qr[v] = sv * ql[v];
          dqr[0][v] = -sv * dql[0][v];
          dqr[1][v] = sv * dql[1][v];
          dqr[2][v] = sv * dql[2][v];
        }
      } else {
        double qb[5];
        farfield_state(vl, n, cfg, qb);
        Vec3 mom{qb[1], qb[2], qb[3]};
        qr[0] = qb[0]; qr[1] = dot(mom, n); qr[2] = dot(mom, t1); qr[3] = dot(mom, t2); qr[4] = qb[4];
        for (int j = 0; j < 3; ++j)
          for (int v = 0; v < 5; ++v) dqr[j][v] = 0.0;
      }
      // R9s (dq0_mode 2): dQ0 = average of the two cells' gradients of Eq. (weno) with the
      // linear weights gamma in place of omega-bar (a side that fell back contributes zero;
      // wall: the mirror of the left one; farfield: zero)
      double dq0s[3][5] = {};
      if (cfg.dq0_mode == 2) {
        double v5[5], g5[5][3], q5[5], dl0[3][5] = {}, dr0[3][5] = {};
        if (!fell_l) {
          weno_point(m, polys[f.owner], f.owner, gp.x, v5, g5, true);
          to_local(v5, g5, q5, dl0);
        }
        if (f.nb >= 0) {
          if (!fell_r) {
            weno_point(m, polys[f.nb], f.nb, sub(gp.x, f.shift), v5, g5, true);
            to_local(v5, g5, q5, dr0);
          }
        } else if (f.bc == kWall) {
          for (int v = 0; v < 5; ++v) {
            double sv = (v >= 1 && v <= 3) ? -1.0 : 1.0;
            dr0[0][v] = -sv * dl0[0][v];
            dr0[1][v] = sv * dl0[1][v];
            dr0[2][v] = sv * dl0[2][v];
          }
        }
        for (int j = 0; j < 3; ++j)
          for (int v = 0; v < 5; ++v) dq0s[j][v] = 0.5 * (dl0[j][v] + dr0[j][v]);
      }
      GpFluxOut o = gks_flux_local(ql, dql, qr, dqr, dt, cfg, cfg.dq0_mode == 2 ? dq0s : nullptr);
      // rotate back to the global frame and accumulate omega_G S F_G
      auto to_global = [&](const double a[5], double out[5]) {
        out[0] = a[0];
        for (int c = 0; c < 3; ++c) out[1 + c] = a[1] * n[c] + a[2] * t1[c] + a[3] * t2[c];
        out[4] = a[4];
      };
      double Fg[5], dFg[5];
      to_global(o.F, Fg);
      to_global(o.dF, dFg);
      for (int v = 0; v < 5; ++v) {
        Fs[v] += gp.wS * Fg[v];
        dFs[v] += gp.wS * dFg[v];
      }
    }
    Ff[fi] = Fs;
    dFf[fi] = dFs;
  }
  if (fallback_count) *fallback_count += fb;
  L.assign((size_t)m.n_cells * 5, 0.0);
  dL.assign((size_t)m.n_cells * 5, 0.0);
  for (int i = 0; i < m.n_cells; ++i) {
    for (int p = 0; p < (int)m.cell_face[i].size(); ++p) {  // local-face order
      int fi = m.cell_face[i][p];
      double sgn = (m.faces[fi].owner == i) ? 1.0 : -1.0;  // outward flux of cell i
      for (int v = 0; v < 5; ++v) {
        L[(size_t)i * 5 + v] -= sgn * Ff[fi][v];
        dL[(size_t)i * 5 + v] -= sgn * dFf[fi][v];
      }
    }
    for (int v = 0; v < 5; ++v) {
      L[(size_t)i * 5 + v] /= m.geom[i].V;
      dL[(size_t)i * 5 + v] /= m.geom[i].V;
    }
  }
}

// Delta t (R6): CFL * min_i h_i / (|U_i| + c_i + 2 nu_i / h_i)
double time_step(const Solver& S, const double* Q) {
  const Mesh& m = S.mesh;
  const Config& cfg = S.cfg;
  double dt = 1e300;
  for (int i = 0; i < m.n_cells; ++i) {
    const double* q = Q + (size_t)i * 5;
    double rho = q[0];
    double u = q[1] / rho, v = q[2] / rho, w = q[3] / rho;
    double p = pressure_of(q, cfg.gamma);
    double c = std::sqrt(cfg.gamma * p / rho);
    double nu = 0.0;
    if (cfg.tau_mode == 1) nu = cfg.mu_inf * std::pow((p / rho) / cfg.t_inf, cfg.mu_exp) / rho;
    double h = m.h_dt[i];
    double dti = cfg.cfl * h / (std::sqrt(u * u + v * v + w * w) + c + 2.0 * nu / h);
    dt = std::min(dt, dti);
  }
  return dt;
}

void s2o4_stage1(int n5, const double* Qn, const double* L, const double* dL, double dt, double* Qs, double* R) {
  for (int k = 0; k < n5; ++k) {
    Qs[k] = Qn[k] + 0.5 * dt * L[k] + 0.125 * dt * dt * dL[k];          // Q*
    R[k] = Qn[k] + dt * L[k] + dt * dt / 6.0 * dL[k];                   // first part of Q^{n+1}
  }
}
void s2o4_stage2(int n5, const double* R, const double* dLs, double dt, double* Qn1) {
  for (int k = 0; k < n5; ++k) Qn1[k] = R[k] + dt * dt / 6.0 * 2.0 * dLs[k];
}

int step(Solver& S, int n_steps, double t_stop, int* done) {
  const int n5 = S.mesh.n_cells * 5;
  std::vector<double> L, dL, Qs(n5), R(n5), dLs, Ls;
  *done = 0;
  for (int s = 0; s < n_steps; ++s) {
    double dt = S.cfg.fixed_dt > 0 ? S.cfg.fixed_dt : time_step(S, S.Q.data());
    bool clipped = false;
    if (t_stop > 0) {
      if (S.t >= t_stop) break;
      if (S.t + dt > t_stop) { dt = t_stop - S.t; clipped = true; }  // land exactly on t_stop
    }
    if (!(dt > 0) || !std::isfinite(dt)) throw OracleError(E_STATE, "non-positive time step");
    residual(S, S.Q.data(), dt, L, dL, &S.fallbacks);
    s2o4_stage1(n5, S.Q.data(), L.data(), dL.data(), dt, Qs.data(), R.data());
    residual(S, Qs.data(), dt, Ls, dLs, &S.fallbacks);
    s2o4_stage2(n5, R.data(), dLs.data(), dt, S.Q.data());
    for (int i = 0; i < S.mesh.n_cells; ++i) {
      const double* q = &S.Q[(size_t)i * 5];
      if (!(q[0] > 0) || !(pressure_of(q, S.cfg.gamma) > 0))
        throw OracleError(E_POSITIVITY, "non-positive density or pressure at cell " + std::to_string(i));
    }
    S.t = clipped ? t_stop : S.t + dt;
    S.last_dt = dt;
    ++*done;
  }
  return 0;
}

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return E_OK;
  } catch (const OracleError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_ARG;
  }
}

Config to_config(const double* c) {
  // flat layout: gamma, cfl, fixed_dt, tau_mode, c1, mu_inf, t_inf, mu_exp, eps, omega_pow, fs[5], dq0_mode, prandtl
  Config k;
  k.gamma = c[0]; k.cfl = c[1]; k.fixed_dt = c[2]; k.tau_mode = (int)c[3]; k.c1 = c[4];
  k.mu_inf = c[5]; k.t_inf = c[6]; k.mu_exp = c[7]; k.eps = c[8]; k.omega_pow = (int)c[9];
  for (int i = 0; i < 5; ++i) k.fs[i] = c[10 + i];
  k.dq0_mode = (int)c[15];
  k.prandtl = c[16];
  if (!(k.prandtl > 0)) throw OracleError(E_ARG, "prandtl must be > 0");
  if (k.dq0_mode < 0 || k.dq0_mode > 2) throw OracleError(E_ARG, "dq0_mode must be 0, 1 or 2");
  return k;
}

}  // namespace

// ============================================================================
// C API (ctypes, oracle/oracle.py)
// ============================================================================
extern "C" {

const char* ora_last_error() { return g_err.c_str(); }

int ora_mesh_create(const double* xyz, int64_t n_nodes, const int8_t* type, const int64_t* cell_nodes, int64_t n_cells,
                    const double* per_origin, const double* per_len, const int64_t* bface_nodes,
                    const int32_t* bface_tag, int64_t n_bf, void** out) {
  return guarded([&] {
    MeshInputC in{xyz, n_nodes, type, cell_nodes, n_cells, per_origin, per_len, bface_nodes, bface_tag, n_bf};
    *out = new Mesh(build_mesh(in));
  });
}
void ora_mesh_destroy(void* h) { delete (Mesh*)h; }

// counts: n_cells, n_faces, n_ghosts, max big stencil, min big stencil, n_subs(max)
void ora_mesh_counts(void* h, int64_t* out) {
  Mesh& m = *(Mesh*)h;
  size_t mx = 0, mn = 1 << 30, ns = 0;
  for (auto& s : m.big) { mx = std::max(mx, s.size()); mn = std::min(mn, s.size()); }
  for (auto& s : m.subs) ns = std::max(ns, s.size());
  out[0] = m.n_cells; out[1] = (int64_t)m.faces.size(); out[2] = m.n_ghosts;
  out[3] = (int64_t)mx; out[4] = (int64_t)mn; out[5] = (int64_t)ns;
}

// geometry of cells and ghosts: V[n], c[n][3], M2[n][9]
void ora_cell_geometry(void* h, double* V, double* c, double* M2) {
  Mesh& m = *(Mesh*)h;
  for (size_t i = 0; i < m.geom.size(); ++i) {
    V[i] = m.geom[i].V;
    for (int a = 0; a < 3; ++a) c[i * 3 + a] = m.geom[i].c[a];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M2[i * 9 + a * 3 + b] = m.geom[i].M2[a][b];
  }
}

// faces: owner, nb (-1 boundary), bc, shift[3], ngp, gp_x[4][3], gp_n[4][3], gp_wS[4]
void ora_faces(void* h, int64_t* owner, int64_t* nb, int32_t* bc, double* shift, int32_t* ngp, double* gx, double* gn,
               double* gw) {
  Mesh& m = *(Mesh*)h;
  for (size_t f = 0; f < m.faces.size(); ++f) {
    const Face& F = m.faces[f];
    owner[f] = F.owner; nb[f] = F.nb; bc[f] = F.bc; ngp[f] = (int)F.gp.size();
    for (int a = 0; a < 3; ++a) shift[f * 3 + a] = F.shift[a];
    for (size_t g = 0; g < F.gp.size(); ++g) {
      for (int a = 0; a < 3; ++a) {
        gx[(f * 4 + g) * 3 + a] = F.gp[g].x[a];
        gn[(f * 4 + g) * 3 + a] = F.gp[g].n[a];
      }
      gw[f * 4 + g] = F.gp[g].wS;
    }
  }
}
void ora_cell_faces(void* h, int64_t* cf /* [n][6], -1 pad */) {
  Mesh& m = *(Mesh*)h;
  for (int i = 0; i < m.n_cells; ++i)
    for (int p = 0; p < 6; ++p) cf[i * 6 + p] = p < (int)m.cell_face[i].size() ? m.cell_face[i][p] : -1;
}
// big stencil of cell i: ids (ghosts >= n_cells) and shifts; returns count
int ora_big_stencil(void* h, int64_t i, int64_t* ids, double* shifts) {
  Mesh& m = *(Mesh*)h;
  const auto& S = m.big[i];
  for (size_t k = 0; k < S.size(); ++k) {
    ids[k] = S[k].id;
    for (int a = 0; a < 3; ++a) shifts[k * 3 + a] = S[k].s[a];
  }
  return (int)S.size();
}
int ora_sub_stencil(void* h, int64_t i, int64_t mm, int64_t* ids) {
  Mesh& m = *(Mesh*)h;
  const auto& S = m.subs[i][mm];
  for (size_t k = 0; k < S.size(); ++k) ids[k] = S[k].id;
  return (int)S.size();
}

// LSQ + WENO of one cell for state Q: P0 coeffs a[9][5], P_m coeffs b[M][3][5],
// beta[M+1][5], wbar[M+1][5]; returns M (or -code on error)
int ora_fit_cell(void* hm, const double* cfgv, const double* Q, int64_t i, double* a, double* b, double* beta,
                 double* wbar) {
  Mesh& m = *(Mesh*)hm;
  int M = -1;
  int rc = guarded([&] {
    Config cfg = to_config(cfgv);
    State st{&m, Q, {}};
    ghost_states(m, cfg, st);
    CellPolys P = fit_cell(m, st, (int)i, cfg);
    M = (int)P.b.size();
    for (int d = 0; d < 9; ++d)
      for (int v = 0; v < 5; ++v) a[d * 5 + v] = P.a[d][v];
    for (int mm = 0; mm < M; ++mm)
      for (int d = 0; d < 3; ++d)
        for (int v = 0; v < 5; ++v) b[(mm * 3 + d) * 5 + v] = P.b[mm][d][v];
    for (int mm = 0; mm <= M; ++mm)
      for (int v = 0; v < 5; ++v) {
        beta[mm * 5 + v] = P.beta[mm][v];
        wbar[mm * 5 + v] = P.wbar[mm][v];
      }
  });
  return rc == E_OK ? M : -rc;
}

// WENO value and gradient of cell i at points x[np][3] (cell i's coordinates)
int ora_weno_points(void* hm, const double* cfgv, const double* Q, int64_t i, int64_t np, const double* x, double* val,
                    double* grad, int linear) {
  Mesh& m = *(Mesh*)hm;
  return guarded([&] {
    Config cfg = to_config(cfgv);
    State st{&m, Q, {}};
    ghost_states(m, cfg, st);
    CellPolys P = fit_cell(m, st, (int)i, cfg);
    for (int64_t k = 0; k < np; ++k) {
      double v5[5], g[5][3];
      weno_point(m, P, (int)i, {x[k * 3], x[k * 3 + 1], x[k * 3 + 2]}, v5, g, linear != 0);
      for (int v = 0; v < 5; ++v) {
        val[k * 5 + v] = v5[v];
        for (int a = 0; a < 3; ++a) grad[(k * 5 + v) * 3 + a] = g[v][a];
      }
    }
  });
}

// moments <u^a>, <v^b>, <w^c> (a < 8) and <xi^{2d}> (d < 3) of one Maxwellian;
// range 0 full, 1 u>0, 2 u<0. prim = rho, U, V, W, lambda
void ora_moments(const double* prim, double K, int range, double* u, double* v, double* w, double* xi) {
  Maxw g{prim[0], prim[1], prim[2], prim[3], prim[4]};
  Moments M = moments_of(g, (Range)range, K);
  for (int k = 0; k < 8; ++k) { u[k] = M.u[k]; v[k] = M.v[k]; w[k] = M.w[k]; }
  for (int k = 0; k < 3; ++k) xi[k] = M.xi[k];
}
// micro-slope: solve sum_j a_j <psi_i psi_j> rho = b_i for a Maxwellian given by conservative q
void ora_micro_slope(const double* q, double K, const double* b, double* a) {
  Maxw g = maxwellian_of(q, K);
  Moments F = moments_of(g, kFull, K);
  micro_slope(F, g.rho, b, a);
}
// full slopes (spatial a[3][5] and temporal A[5]) for a state q and derivatives dq[3][5]
void ora_slopes(const double* q, double K, const double* dq, double* a, double* A) {
  Maxw g = maxwellian_of(q, K);
  Moments F = moments_of(g, kFull, K);
  double d[3][5];
  for (int j = 0; j < 3; ++j)
    for (int v = 0; v < 5; ++v) d[j][v] = dq[j * 5 + v];
  Slopes s = slopes_of(g, F, d);
  for (int j = 0; j < 3; ++j)
    for (int v = 0; v < 5; ++v) a[j * 5 + v] = s.a[j][v];
  for (int v = 0; v < 5; ++v) A[v] = s.A[v];
}
// one Gauss point in the local frame: outputs I_half, I_full, F, dF, Q0 (5 each) and tau
void ora_gp_flux(const double* cfgv, const double* ql, const double* dql, const double* qr, const double* dqr, double dt,
                 double* out) {
  Config cfg = to_config(cfgv);
  double dl[3][5], dr[3][5];
  for (int j = 0; j < 3; ++j)
    for (int v = 0; v < 5; ++v) { dl[j][v] = dql[j * 5 + v]; dr[j][v] = dqr[j * 5 + v]; }
  GpFluxOut o = gks_flux_local(ql, dl, qr, dr, dt, cfg);
  for (int v = 0; v < 5; ++v) {
    out[v] = o.I_half[v]; out[5 + v] = o.I_full[v]; out[10 + v] = o.F[v]; out[15 + v] = o.dF[v]; out[20 + v] = o.Q0[v];
  }
  out[25] = o.tau;
  for (int j = 0; j < 3; ++j)
    for (int v = 0; v < 5; ++v) out[26 + j * 5 + v] = o.dq0[j][v];
}
void ora_local_frame(const double* n, double* t1, double* t2) {
  Vec3 a, b;
  local_frame({n[0], n[1], n[2]}, a, b);
  for (int k = 0; k < 3; ++k) { t1[k] = a[k]; t2[k] = b[k]; }
}
void ora_farfield_state(const double* cfgv, const double* qi, const double* n, double* qb) {
  Config cfg = to_config(cfgv);
  farfield_state(qi, {n[0], n[1], n[2]}, cfg, qb);
}
void ora_s2o4_stage1(int64_t n5, const double* Qn, const double* L, const double* dL, double dt, double* Qs,
                     double* R) {
  s2o4_stage1((int)n5, Qn, L, dL, dt, Qs, R);
}
void ora_s2o4_stage2(int64_t n5, const double* R, const double* dLs, double dt, double* Q) {
  s2o4_stage2((int)n5, R, dLs, dt, Q);
}

int ora_solver_create(void* hm, const double* cfgv, const double* Q0, int threads, void** out) {
  return guarded([&] {
    Solver* S = new Solver();
    S->mesh = *(Mesh*)hm;
    S->cfg = to_config(cfgv);
    S->Q.assign(Q0, Q0 + (size_t)S->mesh.n_cells * 5);
    S->threads = threads > 0 ? threads : 1;
    *out = S;
  });
}
void ora_solver_destroy(void* h) { delete (Solver*)h; }
void ora_solver_set_threads(void* h, int threads) { ((Solver*)h)->threads = threads > 0 ? threads : 1; }
int ora_solver_step(void* h, int n_steps, double t_stop, int* done) {
  Solver& S = *(Solver*)h;
  return guarded([&] { step(S, n_steps, t_stop, done); });
}
void ora_solver_get(void* h, double* Q, double* t, double* last_dt, int64_t* fallbacks) {
  Solver& S = *(Solver*)h;
  std::memcpy(Q, S.Q.data(), S.Q.size() * sizeof(double));
  *t = S.t;
  *last_dt = S.last_dt;
  *fallbacks = S.fallbacks;
}
void ora_solver_set(void* h, const double* Q, double t) {
  Solver& S = *(Solver*)h;
  std::memcpy(S.Q.data(), Q, S.Q.size() * sizeof(double));
  S.t = t;
}
double ora_solver_dt(void* h) {
  Solver& S = *(Solver*)h;
  return time_step(S, S.Q.data());
}
// L(Q), d_t L(Q) for a given state and dt (kernel-level intermediates)
int ora_solver_residual(void* h, const double* Q, double dt, double* L, double* dL, int64_t* fallbacks) {
  Solver& S = *(Solver*)h;
  return guarded([&] {
    std::vector<double> l, dl;
    long long fb = 0;
    residual(S, Q, dt, l, dl, &fb);
    std::memcpy(L, l.data(), l.size() * sizeof(double));
    std::memcpy(dL, dl.data(), dl.size() * sizeof(double));
    *fallbacks = fb;
  });
}
}
