// Internal data model of libhgks (not part of the C-ABI).
//
// Host setup (setup.cpp) turns the caller's node/cell arrays into a
// GlobalMesh (geometry, faces, stencils, least-squares operators) and one
// RankPlan per rank (partition, 3 ghost layers, renumbered device arrays).
// The device runtime (solver.cu) uploads a RankPlan into the caller's
// workspace and runs the kernels (kernels.cuh).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

// P_0 least squares by normal equations with the rows rebuilt on the device from member
// geometry: 1584 -> 944 operator bytes per tet cell (-29 % DRAM bytes of k_recon), but the
// member-geometry gathers make it latency bound: measured on C2 (same box) k_recon 0.422 vs
// 0.433 ms and the step 1.518 vs 1.506 ms (profiles/r02/README.md), so it is built only on
// request (-DHGKS_RECON_NE=1); 0 streams the 9 x K pseudo-inverse
#ifndef HGKS_RECON_NE
#define HGKS_RECON_NE 0
#endif

namespace hgks {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

constexpr int kMaxStencil = 40;  // big-stencil capacity (tet 14-16, hex interior 24)

// Sizes of the per-cell device records for one mesh kind.
struct Layout {
  int cell_type = 4;   // 4 tet, 8 hex, 6 hybrid tet/prism (cells of several kinds, f4)
  int nfaces = 4;      // faces per cell
  int ngp = 3;         // Gauss points per face (R10)
  int nv = 3;          // vertices per face
  int K = 14;          // padded big-stencil width
  int M = 4;           // sub-stencils per cell
  int NM = 6;          // padded members per sub-stencil
  // P_0 part of the per-cell operators: the 9x9 inverse Cholesky factor W of the normal
  // matrix (45 entries + 1 pad, HGKS_RECON_NE) or the K-column pseudo-inverse
  int op0_entries() const { return HGKS_RECON_NE ? 46 : 9 * K; }
  int op_entries() const { return op0_entries() + M * 3 * NM; }
};

struct GlobalMesh {
  int64_t nc = 0;
  std::vector<int8_t> type;
  Layout lay;
  double per_len[3] = {0, 0, 0};
  // cell geometry: V, centroid, second central moments (xx,yy,zz,xy,xz,yz)
  std::vector<double> V, C, M2, h_dt;
  // faces (owner = lower input cell id, normal out of the owner, R19)
  int64_t nf = 0;
  std::vector<int64_t> f_owner, f_nb;   // f_nb = -1 for physical boundary faces
  std::vector<int32_t> f_bc, f_ghost;
  std::vector<double> f_shift;          // [nf][3] neighbour image = neighbour + shift
  std::vector<double> f_vert;           // [nf][4][3] vertices, oriented out of the owner
  std::vector<int8_t> f_nv;             // [nf] vertex count (3 or 4)
  std::vector<double> f_area;
  std::vector<int64_t> cell_face;       // [nc][6]
  // boundary-condition ghosts (one per wall/farfield face)
  int64_t ng = 0;
  std::vector<int64_t> g_cell, g_face;
  std::vector<int32_t> g_bc;
  std::vector<double> gV, gC, gM2, g_normal;
  // stencils: ids >= nc are ghosts (nc + g)
  std::vector<int64_t> nbr_id;          // [nc][6]
  std::vector<double> nbr_shift;        // [nc][6][3]
  std::vector<int64_t> big_off, big_id; // CSR
  std::vector<double> big_shift;
  std::vector<int8_t> sub_slot;         // [nc][M][NM] slot into big stencil, -1 pad
  // (least-squares operators are built per rank for its reconstructed cells:
  //  setup.cpp cell_operators; there is no global table)
  // partition
  int32_t n_ranks = 1;
  // region builds (one rank per process, hgks_mesh_desc.rank_only): cells are the rank's
  // region in ascending global id, gid[k] = global id of region cell k
  int32_t only_rank = -1;
  int64_t nc_global = 0;
  std::vector<int64_t> gid;
  double bbox_lo[3] = {0, 0, 0}, bbox_hi[3] = {0, 0, 0};  // centroid bounding box of the WHOLE mesh
  std::vector<int32_t> part;
  int64_t edge_cut = 0;       // faces between different ranks (after refinement)
  int64_t edge_cut_rcb = 0;   // the same for the plain RCB partition (before refinement)
};

// One kind of face (triangles, quadrilaterals) of a rank's face list: its faces are
// [base, base + n_if + n_wf + n_ff), interior (early ones first), wall, farfield.
struct FaceClass {
  int64_t base = 0, n_if_early = 0, n_if = 0, n_wf = 0, n_ff = 0;
};

// One rank's device-ready arrays.  Local cell order:
//   [ owned (Morton order) | partition ghosts grouped by owner rank |
//     boundary ghosts ]
struct RankPlan {
  int rank = 0;
  int64_t n_owned = 0, n_pghost = 0, n_bghost = 0;
  int64_t ghost_layer[3] = {0, 0, 0};
  int64_t n_local() const { return n_owned + n_pghost + n_bghost; }
  std::vector<int64_t> l2g;             // [n_owned + n_pghost] global ids
  // reconstruction set (recon index order): [early owned | -1 pad to 128 | late owned | layer-1 ghosts]
  int64_t n_recon = 0, n_recon_early = 0, recon_late0 = 0;
  int64_t ld = 0;                       // n_recon padded to the 128-cell tile
  std::vector<int32_t> recon_cell;      // [n_recon] local cell id
  std::vector<int32_t> st_id;           // [K][ld] local ids (entry-major; host only)
  std::vector<int32_t> st_id_tiled;     // same, tiled entry-major (device)
  std::vector<uint8_t> sub_slot;        // [M*NM] per cell, tiled entry-major
  std::vector<uint8_t> st_shift;        // [K] per cell, tiled: periodic image code of each member (HGKS_RECON_NE)
  std::vector<double> cgeo;             // [n_local][10]: centroid (3), M2 (xx,yy,zz,xy,xz,yz), pad (HGKS_RECON_NE)
  std::vector<double> op;               // [op_entries] per cell, tiled entry-major (kernels.cuh k_recon)
  std::vector<double> geo;              // [8] per cell, tiled: V^{2/3}, V^{4/3}, M2 (xx,yy,zz,xy,xz,yz)
  // faces: interior [0, n_if), wall [n_if, n_if + n_wf), farfield after
  // (totals over the face kinds; interior faces [base, base + n_if_early) of a kind need no ghosts)
  int64_t n_faces = 0, n_if = 0, n_if_early = 0, n_wf = 0, n_ff = 0;
  FaceClass fcls[2];                    // triangles, then quadrilaterals
  std::vector<int32_t> f_cells;         // [n_faces][2] local owner / neighbour (bc faces: ghost id)
  std::vector<double> f_geo;            // [n_faces][FG]: nv vertices rel. owner centroid, then d (3)
  int f_geo_stride = 12;
  // update: owned cells
  std::vector<int32_t> cf;              // [nfaces][n_owned] local face id, ~id when not the owner
                                        // (n_faces: a zero row, for cells with fewer faces)
  std::vector<uint8_t> n_sub;           // [ld] sub-stencils per reconstructed cell (hybrid layouts only)
  std::vector<double> inv_v, h_dt;      // [n_owned]
  // boundary ghosts
  std::vector<int32_t> bg_cell, bg_bc;  // [n_bghost]
  std::vector<double> bg_normal;        // [n_bghost][3]
  // exchange plan (per peer)
  std::vector<int32_t> peers;
  std::vector<int64_t> send_off, send_cnt;  // into send_list
  std::vector<int32_t> send_list;           // local owned ids, grouped by peer, global-id order
  std::vector<int64_t> recv_off, recv_cnt;  // local ghost range [recv_off, recv_off + recv_cnt)
  int32_t stencil_min = 0, stencil_max = 0;
  int64_t rank_cut_faces = 0;  // faces of owned cells whose neighbour another rank owns
};

struct MeshDescCopy;

GlobalMesh build_global_mesh(const double* xyz, int64_t n_nodes, const int8_t* type, const int64_t* cell_nodes,
                             int64_t n_cells, const double* per_origin, const double* per_len,
                             const int64_t* bface_nodes, const int32_t* bface_tag, int64_t n_bf, int32_t n_ranks,
                             const int32_t* cell_part, int32_t rank_only);
RankPlan build_rank_plan(const GlobalMesh& gm, int rank);

}  // namespace hgks
