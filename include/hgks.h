/*
 * hgks.h -- C-ABI of the B200-native HGKS hot path (libhgks.so).
 *
 * The library advances the high-order gas-kinetic scheme of Wang, Cao & Pan,
 * arXiv 2407.00656 (PAPER.md, cited "P:n"), on tetrahedral, hexahedral and hybrid
 * tetrahedral/prismatic unstructured meshes, on one CUDA device per process:
 *   - third-order WENO reconstruction per cell      (Eqs. polys/weno)
 *   - BGK gas-kinetic flux per face Gauss point      (Eqs. flux-G/flux)
 *   - two-stage fourth-order update + CFL minimum    (Alg. 2)
 *   - halo exchange of 3 ghost layers + min(dt), NCCL
 * Readings of points where the paper is silent are DESIGN.md R1-R30.
 *
 * Conventions for every call:
 *   - Return value: HGKS_OK (0) or an error code below; nothing throws or
 *     aborts across this ABI.  hgks_last_error() returns a thread-local,
 *     NUL-terminated message naming the offending cell/face when relevant.
 *   - Host pointers are plain caller-owned arrays; the library deep-copies
 *     what it keeps.  Device memory is owned by the CALLER: it allocates a
 *     workspace of hgks_workspace_size() bytes (e.g. a torch uint8 CUDA
 *     tensor) and passes its pointer to hgks_init; the library carves all its
 *     device arrays from it and never calls cudaMalloc on the hot path.
 *   - `stream` is a cudaStream_t of the current device (NULL = legacy
 *     default stream).  All kernels run on it; calls return once the work is
 *     enqueued unless they must read a device value (documented per call).
 *   - Conserved variables are Q = (rho, rhoU, rhoV, rhoW, rhoE),
 *     host layout [n][5] row-major (AoS), fp64.
 */
#ifndef HGKS_H_
#define HGKS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hgks_status;
#define HGKS_OK 0
#define HGKS_E_ARG 1        /* invalid argument / call order */
#define HGKS_E_MESH 2       /* degenerate cell, non-manifold face, unsupported element, unmatched face */
#define HGKS_E_STENCIL 3    /* rank-deficient least-squares stencil */
#define HGKS_E_CUDA 4       /* CUDA runtime error */
#define HGKS_E_NCCL 5       /* NCCL error or NCCL unavailable for n_ranks > 1 */
#define HGKS_E_POSITIVITY 6 /* non-positive density or pressure after an update */
#define HGKS_E_STATE 7      /* dt <= 0 / non-finite state */

#define HGKS_TET 4
#define HGKS_PRISM 6        /* triangular prism (wedge); mixes with tets only (R30) */
#define HGKS_HEX 8
#define HGKS_BC_WALL 1      /* no-slip adiabatic wall (R25) */
#define HGKS_BC_FARFIELD 2  /* Riemann-invariant inlet/outlet (R25) */

typedef struct hgks_mesh hgks_mesh;
typedef struct hgks_solver hgks_solver;

/* Mesh description.  All arrays are read during hgks_mesh_create only. */
typedef struct {
  const double* xyz;          /* [n_nodes][3] node coordinates */
  int64_t n_nodes;
  const int8_t* cell_type;    /* [n_cells] all HGKS_HEX, or any mix of HGKS_TET and HGKS_PRISM
                                 (other mixes: HGKS_E_MESH) */
  const int64_t* cell_nodes;  /* [n_cells][8], -1 padded; tet: 4 nodes, face p opposite node p
                                 (P:541-549); hex: VTK order, faces 0/5 = (0123)/(4567) (R17);
                                 prism: VTK wedge order, triangles (012)/(345), sides (0143),
                                 (1254), (2035) (R30) */
  int64_t n_cells;
  double periodic_origin[3];  /* periodic box; length 0 along an axis = not periodic (R23) */
  double periodic_length[3];
  const int64_t* bface_nodes; /* [n_bfaces][4], -1 padded: physical boundary faces */
  const int32_t* bface_tag;   /* [n_bfaces] HGKS_BC_WALL / HGKS_BC_FARFIELD */
  int64_t n_bfaces;
  int32_t n_ranks;            /* >= 1; > 1 builds the k-way partition + 3 ghost layers */
  const int32_t* cell_part;   /* optional [n_cells] rank of every cell (external partition), or NULL */
  int32_t rank_only;          /* 0: build the whole mesh and the plans of every rank (one process per
                                 group: loopback, tests, tools); r + 1 (n_ranks > 1): build only rank
                                 r's region -- its owned cells and four node layers around them --
                                 so host memory and time are O(owned + ghosts) per process, apart from
                                 one pass over the cell list (centroids, partition: 28 B per cell).
                                 Calls for other ranks then fail with HGKS_E_ARG; edge_cut is -1
                                 (rank_cut_faces of each rank sum to twice the global cut); the
                                 partition is plain RCB (the boundary refinement needs the whole
                                 face graph), so it may differ from a rank_only = 0 build. */
} hgks_mesh_desc;

/* Solver configuration (readings R4, R6, R7, R13, R14, R24). */
typedef struct {
  double gamma;        /* specific-heat ratio (K = (5-3 gamma)/(gamma-1)) */
  double cfl;          /* dt = cfl * min_i h_i / (|U_i| + c_i + 2 nu_i / h_i)  (R6) */
  double fixed_dt;     /* > 0: use this dt every step instead of the CFL rule */
  int32_t tau_mode;    /* 0: tau = 0 (smooth flows); 1: tau = mu/p + c1 |pl-pr|/(pl+pr) dt */
  double c1;
  double mu_inf, t_inf, mu_exp;  /* mu = mu_inf (T / t_inf)^mu_exp, T = p/rho */
  double eps;          /* WENO epsilon */
  int32_t omega_pow;   /* 1 (as printed) or 2 */
  double freestream[5];/* rho, U, V, W, p for farfield faces */
  int32_t precision;   /* working precision of the hot path: 64 (fp64, the parity path) or 32
                          (the FP32 variant; the CFL bound, time and the caller's
                          state arrays stay fp64).  Anything else: HGKS_E_ARG from hgks_init. */
  int32_t dq0_mode;    /* equilibrium slopes dQ0 (P:306-308 prints only <a-bar> = dQ0/dn):
                          0 = average of the two reconstructed gradients (R9, default),
                          1 = kinetic weighting rho_l<a^l psi>_{u>0} + rho_r<a^r psi>_{u<0} (R9k),
                          2 = average of the two cells' linear-weight (P_0) gradients (R9s; adds a
                              second 50-value record per cell to the workspace).
                          1 and 2 need precision 64 (HGKS_E_ARG otherwise). */
  double prandtl;      /* Prandtl number of the heat-flux correction (R29; P:1203-1210 runs the viscous
                          sphere): the energy flux gains (1/Pr - 1) x the heat flux of the
                          non-equilibrium part of Eq. (flux) (zero for tau_mode 0).  0 or 1 = no
                          correction (BGK, Pr = 1); needs precision 64 and dq0_mode 0. */
} hgks_config;

#define HGKS_TRANSPORT_NCCL 0      /* one process per GPU, NCCL send/recv + allreduce */
#define HGKS_TRANSPORT_LOOPBACK 1  /* all ranks in one process on one device, advanced together by
                                      hgks_group_step (exchange = fused put k_put: send rows written
                                      straight into the receivers' ghost rows); for testing the
                                      partitioned path on a single GPU */
#define HGKS_TRANSPORT_P2P 2       /* one process per GPU on one node: halo by the fused put k_put
                                      into the peers' ghost rows over NVLink (CUDA IPC, per-stage
                                      epoch flags; hgks_p2p_export/connect), dt by NCCL allreduce */
#define HGKS_P2P_HANDLE_BYTES 448

/* Distributed context. */
typedef struct {
  int32_t rank, n_ranks;
  int32_t device;            /* CUDA ordinal used by this rank */
  int32_t transport;         /* HGKS_TRANSPORT_* */
  uint8_t nccl_id[128];      /* ncclUniqueId created by rank 0, broadcast by the caller (NCCL only) */
} hgks_dist;

typedef struct {
  int64_t n_cells_global;
  int64_t n_owned;           /* cells updated by this rank */
  int64_t n_ghost;           /* partition ghosts (3 layers) */
  int64_t ghost_layer[3];
  int64_t n_bghost;          /* boundary-condition ghosts (one per wall/farfield face) */
  int64_t n_faces;           /* faces whose flux this rank computes */
  int64_t n_faces_bc;        /* ... of which wall/farfield faces */
  int32_t stencil_min, stencil_max;  /* big stencil sizes over owned cells (self excluded) */
  int32_t n_sub;             /* sub-stencils per cell (4 tet, 8 hex; hybrid meshes: 6, the most a
                                 cell has -- prisms 6, tets 4) */
  int32_t n_peers;           /* ranks this rank exchanges ghosts with */
  int64_t send_cells, recv_cells;    /* per stage */
  int64_t edge_cut;          /* faces between different ranks (global; RCB + FM boundary refinement);
                                -1 for a rank_only build */
  int64_t n_early_cells;     /* owned cells reconstructed while the halo exchange is in flight */
  int64_t n_early_faces;     /* interior faces fluxed while the halo exchange is in flight */
  int64_t edge_cut_rcb;      /* faces between different ranks of the plain RCB partition, before the
                                boundary refinement (equal to edge_cut for a caller partition) */
  int64_t rank_cut_faces;    /* faces of this rank's owned cells whose neighbour another rank owns */
} hgks_mesh_stats;

typedef struct {
  int64_t steps_done;        /* steps with dt > 0 performed by this call */
  double t;                  /* simulation time after the call */
  double last_dt;
  int64_t fallbacks;         /* cumulative positivity fallbacks at Gauss points (R21) */
} hgks_step_info;

/* Build geometry, faces, periodic pairing, stencils (Alg. 1), least-squares
 * operators, locality (Morton) renumbering and, for n_ranks > 1, the
 * partition with 3 ghost layers and per-peer send/receive plans.  Host only. */
hgks_status hgks_mesh_create(const hgks_mesh_desc* desc, hgks_mesh** out);
hgks_status hgks_mesh_destroy(hgks_mesh* mesh);
hgks_status hgks_mesh_info(const hgks_mesh* mesh, int32_t rank, hgks_mesh_stats* out);

/* Device bytes rank `rank` needs for `cfg`. */
hgks_status hgks_workspace_size(const hgks_mesh* mesh, const hgks_config* cfg, int32_t rank, size_t* bytes);

/* Upload the mesh data of this rank into the caller's workspace and set the
 * initial state h_Q0 ([n_cells_global][5], caller's cell order; each rank
 * takes its own cells).  dist may be NULL for a single process.  Synchronous
 * with respect to `stream` (returns after the uploads completed). */
hgks_status hgks_init(const hgks_mesh* mesh, const hgks_config* cfg, const hgks_dist* dist, void* d_workspace,
                      size_t workspace_bytes, void* stream, const double* h_Q0, hgks_solver** out);
hgks_status hgks_destroy(hgks_solver* solver);

/* Advance up to n_steps S2O4 steps (Alg. 2).  If t_stop > 0 the last step is
 * clipped to land exactly on t_stop and no step starts at t >= t_stop.  The
 * time step is kept on the device (no host synchronisation) unless `info` is
 * non-NULL, in which case the call synchronises and fills it; positivity
 * failures are reported only then (HGKS_E_POSITIVITY, cell id in the message).
 * A step past t_stop (t >= t_stop) has dt = 0 and leaves the state unchanged.
 * HGKS_E_STATE for n_steps > 0 on a HGKS_TRANSPORT_LOOPBACK solver of a group with
 * n_ranks > 1 (its ghosts are filled only by hgks_group_step; n_steps = 0 with info
 * only synchronises and reports) and for a HGKS_TRANSPORT_P2P
 * solver before hgks_p2p_connect. */
hgks_status hgks_step(hgks_solver* solver, int32_t n_steps, double t_stop, hgks_step_info* info);

/* Replace the state (host [n_cells_global][5], caller order) and time.  Used
 * for restart and for end-to-end timing.  Asynchronous on the stream (the host
 * buffer must stay valid until the stream reaches this point; pinned memory
 * recommended). */
hgks_status hgks_set_state(hgks_solver* solver, const double* h_Q, double t);

/* Copy this rank's owned cells into h_Q ([n_owned][5]) in the caller's input
 * order (ascending global id); h_gid (optional, [n_owned]) receives the global
 * ids; t (optional) the time.  Synchronises the stream. */
hgks_status hgks_get_state(const hgks_solver* solver, double* h_Q, int64_t* h_gid, double* t);

/* Pipelined host I/O.  hgks_set_state copies on an internal H2D stream into one of
 * two device staging slots and the solver stream waits for it; hgks_get_state_async
 * enqueues the gather of the current state on the solver stream and the D2H into
 * h_Q ([n_owned][5], ascending global id) on an internal D2H stream, and returns
 * at once.  So the copies of step k+1's input and of step k's result overlap the
 * compute of neighbouring steps (both directions at once).  h_Q is valid, and the
 * buffers given to either call may be reused, after hgks_sync (pinned host memory
 * is needed for the copies to be asynchronous).  At most two results may be in
 * flight: a third hgks_get_state_async waits on the device for the first D2H. */
hgks_status hgks_get_state_async(hgks_solver* solver, double* h_Q);
hgks_status hgks_sync(hgks_solver* solver);

/* Parity intermediates (single rank): L(Q) and d_t L(Q)
 * for state h_Q at step dt, [n_cells][5] caller order each.  Synchronous. */
hgks_status hgks_debug_residual(hgks_solver* solver, const double* h_Q, double dt, double* h_L, double* h_dL);

/* Per-kernel device time: when enabled, every kernel launch is bracketed by
 * CUDA events on the solver stream.  hgks_kernel_times fills up to `cap`
 * entries of (name, timed launches, total milliseconds over exactly those
 * launches) and returns the count in *n.
 * Synchronises the stream. */
hgks_status hgks_set_profiling(hgks_solver* solver, int32_t enabled);
hgks_status hgks_kernel_times(hgks_solver* solver, int32_t cap, char (*names)[32], int64_t* launches,
                              double* total_ms, int32_t* n);
/* Loopback transport: advance the solvers of ranks 0..n-1 (created with
 * HGKS_TRANSPORT_LOOPBACK on one device and stream, in rank order) by n_steps
 * S2O4 steps, exchanging ghosts by the fused put (one k_put per sending rank and stage,
 * P:856-869) and reducing min(dt) exactly.  The first call uploads each rank's
 * (receiver, row) put map (synchronous); later calls are asynchronous on the
 * shared stream. */
hgks_status hgks_group_step(hgks_solver* const* solvers, int32_t n, int32_t n_steps, double t_stop);

/* Fused halo put map of rank `rank` (host; the loopback group's k_put
 * uses it): for send row j (the order of hgks_mesh_plan's send_list), the receiving
 * rank recv_rank[j] and the local ghost row recv_row[j] there that takes the cell's
 * state.  Arrays of send_cells entries, caller-allocated.  HGKS_E_STATE if two ranks'
 * plans disagree, HGKS_E_ARG on a NULL pointer or a rank out of range. */
hgks_status hgks_mesh_put_map(const hgks_mesh* mesh, int32_t rank, int32_t* recv_rank, int32_t* recv_row);

/* Export rank `rank`'s partition plan (host, for tests and tools): l2g
 * [n_owned + n_ghost] global ids of the local cells (owned first), peers
 * [n_peers], per-peer send offsets/counts into send_list [send_cells] (local
 * owned ids, the owner's global-id order) and receive ranges [recv_off,
 * recv_off + recv_cnt) of local ghost ids.  Any pointer may be NULL. */
hgks_status hgks_mesh_plan(const hgks_mesh* mesh, int32_t rank, int64_t* l2g, int32_t* peers, int64_t* send_off,
                           int64_t* send_cnt, int32_t* send_list, int64_t* recv_off, int64_t* recv_cnt);

/* Create the 128-byte NCCL unique id on one rank (to be broadcast by the caller,
 * e.g. over torch.distributed, and passed in hgks_dist.nccl_id).  Host only. */
hgks_status hgks_nccl_unique_id(uint8_t* out);

/* HGKS_TRANSPORT_P2P setup.  Every rank calls
 * hgks_p2p_export after hgks_init to write HGKS_P2P_HANDLE_BYTES describing its
 * workspace (a CUDA IPC handle of the allocation, offsets of the state rows and of the
 * epoch flags); the caller all-gathers the blobs (rank order, n_ranks x
 * HGKS_P2P_HANDLE_BYTES) and every rank calls hgks_p2p_connect with them, which maps
 * the peers' workspaces and uploads the put map.  hgks_step fails with HGKS_E_STATE
 * before the connect.  Each stage then puts the send rows into the receivers' ghost
 * rows, releases an epoch flag to each receiver and acquires the senders' flags before
 * its ghost-dependent work; receivers release "consumed" after the stage so the next
 * put never overwrites rows still being read.  Needs one GPU per rank with peer access
 * (HGKS_E_ARG / HGKS_E_CUDA otherwise).  Validated by the plan tests and the loopback
 * group's k_put; the cross-process flag protocol needs a multi-GPU node to exercise. */
/* Diagnostic on the current device, no peers: k_put through a pointer table into a
 * second buffer (rows checked bitwise), k_p2p_signal on two flags (read back), then
 * k_p2p_wait on flags that already hold the epoch.  HGKS_E_CUDA with a message on any
 * mismatch. */
hgks_status hgks_p2p_selftest(void);
hgks_status hgks_p2p_export(const hgks_solver* solver, uint8_t* out);
hgks_status hgks_p2p_connect(hgks_solver* solver, const uint8_t* blobs);

/* Diagnostic of the NCCL transport on the current device: a one-rank communicator
 * does exactly the calls a multi-rank step makes (grouped ncclSend/ncclRecv of
 * fp64 and fp32 halo buffers, here to itself, and the uint64 ncclAllReduce(min) of
 * the CFL bound) and checks the results.  HGKS_E_NCCL with a message on failure. */
hgks_status hgks_nccl_selftest(void);

/* Number of kernels launched by this solver so far (all kinds). */
hgks_status hgks_launch_count(const hgks_solver* solver, int64_t* launches);

const char* hgks_last_error(void);
const char* hgks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HGKS_H_ */
