// Device runtime and C-ABI of libhgks (include/hgks.h).
//
// One solver per process/GPU.  The caller owns device memory (a workspace
// carved here) and the stream; NCCL (loaded at run time with dlopen, only when
// n_ranks > 1) carries the per-stage halo exchange on a comm stream, overlapped
// with the ghost-free half of every stage, and the per-step min(dt).  On one
// rank a step is replayed from a captured CUDA graph; host state copies run on
// two internal copy streams, double-buffered (hgks_get_state_async).  The hot
// path is compiled for fp64 (p64) and fp32 (p32) and dispatched per solver.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/hgks.h"
#include "internal.h"
#include "kernels.cuh"

using namespace hgks;

// ============================================================================
// errors
// ============================================================================
static thread_local std::string g_last_error;

#define CUDA_TRY(x)                                                                                    \
  do {                                                                                                 \
    cudaError_t e_ = (x);                                                                              \
    if (e_ != cudaSuccess) throw Error(HGKS_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class F>
static hgks_status guard(F&& f) {
  try {
    f();
    return HGKS_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HGKS_E_ARG;
  } catch (...) {
    g_last_error = "unknown error";
    return HGKS_E_ARG;
  }
}

// ============================================================================
// NCCL, resolved at run time (no link-time dependency for single-GPU use)
// ============================================================================
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { ncclUint64 = 5, ncclFloat32 = 7, ncclFloat64 = 8 };
enum { ncclMin = 3 };
struct Nccl {
  void* h = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.Send = (decltype(n.Send))dlsym(n.h, "ncclSend");
    n.Recv = (decltype(n.Recv))dlsym(n.h, "ncclRecv");
    n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
    n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
  });
  return n;
}
#define NCCL_TRY(x)                                                                                              \
  do {                                                                                                           \
    int r_ = (x);                                                                                                \
    if (r_ != 0)                                                                                                 \
      throw Error(HGKS_E_NCCL, std::string(#x) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r_) : "")); \
  } while (0)
}  // namespace

// ============================================================================
// mesh handle
// ============================================================================
struct hgks_mesh {
  GlobalMesh gm;
  std::map<int, std::unique_ptr<RankPlan>> plans;
  std::mutex mu;
  const RankPlan& plan(int rank) {
    std::lock_guard<std::mutex> lk(mu);
    if (rank < 0 || rank >= gm.n_ranks) throw Error(HGKS_E_ARG, "rank out of range");
    auto it = plans.find(rank);
    if (it == plans.end()) it = plans.emplace(rank, std::make_unique<RankPlan>(build_rank_plan(gm, rank))).first;
    return *it->second;
  }
};

// ============================================================================
// workspace layout
// ============================================================================
namespace {
struct Carve {
  char* base;
  size_t off = 0, cap;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    size_t bytes = n * sizeof(T);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += bytes;
    if (base && off > cap) throw Error(HGKS_E_ARG, "workspace too small");
    return p;
  }
};

int round32(int64_t n) { return (int)((n + 31) / 32 * 32); }

struct DevArrays {
  // working-precision arrays (double for fp64, float for fp32)
  void *Q, *Qtmp, *R, *ceff, *ceff0, *F1, *F2, *op, *geo, *cgeo, *f_geo, *inv_v, *h_dt, *bg_normal, *sendbuf;
  double *stage_in[2], *stage_out[2];  // caller-order staging (fp64), double-buffered for pipelining
  int *recon_cell, *st_id, *f_cells, *cf, *bg_cell, *bg_bc, *send_list, *out_local;
  int2* put_dst;  // fused halo put: (receiver rank, receiver row) per send row (f3)
  P2PFlags* flags;  // cross-process put: epoch flags written by the peers (f3)
  int64_t* in_row;
  uint8_t* sub_slot;
  uint8_t* n_sub;  // sub-stencils per reconstructed cell (hybrid layouts), else null
  uint8_t* st_shift;
  Ctrl* ctrl;
};

// rs = bytes of the working precision; dq0_mode 2 (R9s) adds the P_0 records
size_t layout(const GlobalMesh& gm, const RankPlan& rp, size_t rs, int dq0_mode, Carve& c, DevArrays& d) {
  const Layout& L = gm.lay;
  const size_t nq = (size_t)QS * round32(rp.n_local());
  const int64_t ncl = rp.n_owned + rp.n_pghost;
  auto R = [&](size_t n) { return (void*)c.take<char>(n * rs); };
  // experiment knobs (address-mapping study): extra bytes before the records and before the
  // operators, in KiB (HGKS_PAD_REC, HGKS_PAD_OP; default 0)
  auto pad_kib = [](const char* name) -> size_t {
    const char* e = std::getenv(name);
    return e ? (size_t)std::strtoull(e, nullptr, 10) * 1024 : 0;
  };
  d.ctrl = c.take<Ctrl>(1);
  d.Q = R(nq);
  d.Qtmp = R(nq);
  d.R = R((size_t)QS * rp.n_owned);
  c.off += pad_kib("HGKS_PAD_REC");
  d.ceff = R((size_t)kRec * ncl);
  d.ceff0 = dq0_mode == 2 ? R((size_t)kRec * ncl) : nullptr;
  // one zero row past the last face: the update's entry for a face a cell does not have
  d.F1 = R((size_t)10 * (rp.n_faces + 1));
  d.F2 = R((size_t)5 * (rp.n_faces + 1));
  d.recon_cell = c.take<int>(rp.n_recon);
  d.st_id = c.take<int>((size_t)L.K * rp.ld);
  d.sub_slot = c.take<uint8_t>((size_t)L.M * L.NM * rp.ld);
  d.n_sub = rp.n_sub.empty() ? nullptr : c.take<uint8_t>(rp.n_sub.size());
  c.off += pad_kib("HGKS_PAD_OP");
  d.op = R((size_t)L.op_entries() * rp.ld);
  d.geo = R((size_t)8 * rp.ld);
  d.st_shift = c.take<uint8_t>(HGKS_RECON_NE ? (size_t)L.K * rp.ld : 1);
  d.cgeo = R(HGKS_RECON_NE ? (size_t)10 * rp.n_local() : 1);
  d.f_cells = c.take<int>((size_t)2 * rp.n_faces);
  d.f_geo = R((size_t)rp.f_geo_stride * rp.n_faces);
  d.cf = c.take<int>((size_t)L.nfaces * rp.n_owned);
  d.inv_v = R(rp.n_owned);
  d.h_dt = R(rp.n_owned);
  d.bg_cell = c.take<int>(std::max<int64_t>(1, rp.n_bghost));
  d.bg_bc = c.take<int>(std::max<int64_t>(1, rp.n_bghost));
  d.bg_normal = R(std::max<int64_t>(3, 3 * rp.n_bghost));
  d.send_list = c.take<int>(std::max<size_t>(1, rp.send_list.size()));
  d.sendbuf = R(std::max<size_t>(QS, QS * rp.send_list.size()));
  d.put_dst = c.take<int2>(std::max<size_t>(1, rp.send_list.size()));
  d.flags = c.take<P2PFlags>(1);
  d.out_local = c.take<int>(rp.n_owned);
  d.in_row = c.take<int64_t>(rp.n_owned);
  // staging for set/get_state: single rank copies the caller's whole array
  const int64_t n_in = gm.n_ranks == 1 ? gm.nc : rp.n_owned;
  for (int k = 0; k < 2; ++k) {
    d.stage_in[k] = c.take<double>((size_t)5 * n_in);
    d.stage_out[k] = c.take<double>((size_t)5 * rp.n_owned);
  }
  return c.off + 256;
}
}  // namespace

// ============================================================================
// solver
// ============================================================================
struct KStat {
  int64_t launches = 0;       // all launches
  int64_t timed = 0;          // launches bracketed by profiling events (ms covers exactly these)
  double ms = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};

struct hgks_solver {
  hgks_mesh* mesh;
  const RankPlan* rp;
  Layout lay;
  hgks_config cfg;
  GasParams gp;
  bool fp32 = false;  // working precision of the hot path (FP32 variant)
  int recon_pair = -1;  // two lanes per reconstructed cell: -1 = measured choice (fp32 tets only:
                        // -7 %; slower for fp64 and for fp32 hexes), HGKS_RECON_PAIR=0/1 forces
  size_t rs = sizeof(double);
  int rank = 0, n_ranks = 1, device = 0, transport = HGKS_TRANSPORT_NCCL;
  size_t recon_smem_set = 0;
  int recon_t1 = 0;  // end tile of the current reconstruction launch
  cudaStream_t comm_stream = nullptr;  // NCCL halo exchange (overlapped with the early work)
  cudaEvent_t ev_packed = nullptr, ev_halo = nullptr;
  // min(dt) allreduce on the comm stream (n_ranks > 1): issued after k_update2, waited for
  // only where the next step first needs dt (hidden behind stage-1 work)
  cudaEvent_t ev_upd2 = nullptr, ev_dt = nullptr;
  bool dt_pending = false;     // an allreduce is in flight on the comm stream
  bool begin_pending = false;  // this step's k_step_begin is deferred until dt is needed
  double cur_t_stop = 0.0;
  bool put_ready = false;  // put_dst uploaded (loopback group, first hgks_group_step)
  // HGKS_TRANSPORT_P2P: peers' workspaces mapped by CUDA IPC (hgks_p2p_connect)
  bool p2p_ready = false;
  unsigned long long epoch = 0;  // stage counter, identical on every rank
  void* peer_base[kMaxGroup] = {};
  void* peer_Q[kMaxGroup] = {};
  P2PFlags* peer_flags[kMaxGroup] = {};
  std::vector<int> put_to, recv_from;  // receivers of this rank's puts, senders into it
  cudaStream_t stream = nullptr;
  DevArrays d{};
  size_t nq = 0;  // values in Q
  ncclComm_t comm = nullptr;
  int64_t launches = 0;
  bool profiling = false;
  std::map<std::string, KStat> kstat;
  std::vector<int> peers;
  std::vector<double> host_stage;  // multi-rank set_state gather
  double* pinned[2] = {nullptr, nullptr};  // multi-rank set_state gather (one per staging slot)
  // host<->device pipelining (hgks_set_state / hgks_get_state_async): copies run on their
  // own streams, double-buffered, ordered against the compute stream by events
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_scattered[2] = {}, ev_gathered[2] = {}, ev_d2h[2] = {};
  int in_slot = 0, out_slot = 0;
  // CUDA graph of one full step (single rank, profiling off): captured on an internal
  // stream, replayed on the solver stream; re-captured when t_stop changes
  bool use_graphs = true;  // HGKS_GRAPHS=0 disables
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t step_graph = nullptr;
  double graph_t_stop = 0.0;
  int64_t graph_launches = 0;  // kernel launches per replay
  int64_t eager_steps = 0;
  std::vector<cudaEvent_t> event_pool;  // reusable profiling events
};

namespace {

void record_launch(hgks_solver* s, const char* name, cudaEvent_t a, cudaEvent_t b) {
  KStat& k = s->kstat[name];
  k.launches++;
  if (a) {
    k.timed++;
    k.pending.push_back({a, b});
  }
}

cudaEvent_t pooled_event(hgks_solver* s) {
  if (s->event_pool.empty()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      s->event_pool.push_back(e);
    }
  }
  cudaEvent_t e = s->event_pool.back();
  s->event_pool.pop_back();
  return e;
}

template <class Launch>
void launch(hgks_solver* s, const char* name, Launch&& fn) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (s->profiling) {
    a = pooled_event(s);
    b = pooled_event(s);
    CUDA_TRY(cudaEventRecord(a, s->stream));
  }
  fn();
  CUDA_TRY(cudaGetLastError());
  if (s->profiling) CUDA_TRY(cudaEventRecord(b, s->stream));
  s->launches++;
  record_launch(s, name, a, b);
}

inline int blocks(int64_t n, int b) { return (int)((n + b - 1) / b); }

template <class L>
typename L::GasT make_gas_for(const GasParams& g) {
  return L::gas(g);
}

template <class L, class T>
typename L::RealT* as(T* p) {
  return reinterpret_cast<typename L::RealT*>(const_cast<void*>(static_cast<const void*>(p)));
}

template <class L, int K, int M, int NM>
void run_recon_k(hgks_solver* s, const typename L::ReconArgsT& a) {
  // hybrid layouts (NM = 7, per-cell sub-stencil counts) have the one-lane kernel only
  constexpr bool kPair = NM != 7;
  if (!s->recon_smem_set) {  // one reconstruction instantiation per solver (K, M, NM, precision fixed)
    CUDA_TRY((L::template recon_smem<K, M, NM>()));
    if constexpr (kPair) CUDA_TRY((L::template recon_pair_smem<K, M, NM>()));
    s->recon_smem_set = 1;
  }
  const int n_tiles = s->recon_t1 - a.tile0;
  if (n_tiles <= 0) return;
  if constexpr (kPair) {
    if (s->recon_pair == 1 || (s->recon_pair < 0 && s->fp32 && K <= 16)) {
      launch(s, "k_recon", [&] { L::template recon_pair<K, M, NM>(n_tiles, s->stream, a); });
      return;
    }
  }
  launch(s, "k_recon", [&] { L::template recon<K, M, NM>(n_tiles, s->stream, a); });
}

// part 0: tiles of the early cells, 1: the rest, 2: all
template <class L>
void run_recon(hgks_solver* s, const void* Q, int part) {
  const Layout& LY = s->lay;
  const RankPlan& rp = *s->rp;
  typename L::ReconArgsT a;
  a.Q = as<L>(Q);
  a.n_recon = (int)rp.n_recon;
  const int t_mid = (int)(rp.recon_late0 / kTile), t_end = (int)((rp.n_recon + kTile - 1) / kTile);
  a.tile0 = part == 1 ? t_mid : 0;
  s->recon_t1 = part == 0 ? t_mid : t_end;
  a.ld = (int)s->rp->ld;
  a.recon_cell = s->d.recon_cell;
  a.st_id = s->d.st_id;
  a.sub_slot = s->d.sub_slot;
  a.n_sub = s->d.n_sub;
  a.st_shift = s->d.st_shift;
  a.cgeo = as<L>(s->d.cgeo);
  for (int k = 0; k < 3; ++k) a.per_len[k] = (typename L::RealT)s->mesh->gm.per_len[k];
  a.op = as<L>(s->d.op);
  a.geo = as<L>(s->d.geo);
  a.ceff = as<L>(s->d.ceff);
  a.ceff0 = s->d.ceff0 ? as<L>(s->d.ceff0) : nullptr;
  a.eps = (typename L::RealT)s->cfg.eps;
  a.omega_pow = s->cfg.omega_pow;
  if (LY.cell_type == 6) {  // hybrid tet/prism (f4): 6 sub-stencils of up to 7 members, K >= 20
    switch (LY.K) {
      case 20: run_recon_k<L, 20, 6, 7>(s, a); break;
      case 24: run_recon_k<L, 24, 6, 7>(s, a); break;
      case 32: run_recon_k<L, 32, 6, 7>(s, a); break;
      default: run_recon_k<L, 40, 6, 7>(s, a); break;
    }
  } else if (LY.cell_type == 4) {
    switch (LY.K) {
      case 14: run_recon_k<L, 14, 4, 6>(s, a); break;
      case 16: run_recon_k<L, 16, 4, 6>(s, a); break;
      case 20: run_recon_k<L, 20, 4, 6>(s, a); break;
      case 24: run_recon_k<L, 24, 4, 6>(s, a); break;
      case 32: run_recon_k<L, 32, 4, 6>(s, a); break;
      default: run_recon_k<L, 40, 4, 6>(s, a); break;
    }
  } else {
    switch (LY.K) {
      case 14: run_recon_k<L, 14, 8, 3>(s, a); break;
      case 16: run_recon_k<L, 16, 8, 3>(s, a); break;
      case 20: run_recon_k<L, 20, 8, 3>(s, a); break;
      case 24: run_recon_k<L, 24, 8, 3>(s, a); break;
      case 32: run_recon_k<L, 32, 8, 3>(s, a); break;
      default: run_recon_k<L, 40, 8, 3>(s, a); break;
    }
  }
}

template <class L, int NV, int BC, int DQ0, bool PR = false>
void launch_flux_q(hgks_solver* s, const typename L::FluxArgsT& a, int stage, bool tau0) {
  constexpr int NGP = NV == 3 ? 3 : 4, B = NGP * HGKS_FLUX_FPB;
  // faces per block: NGP lanes per face, or 10 faces per warp with the shuffle reduction
  constexpr int FPBk = HGKS_FLUX_WARPRED ? (B / 32) * (32 / NGP) : B / NGP;
  const int nb = (int)((a.n_faces + FPBk - 1) / FPBk);
  const char* names[2][2] = {{"k_flux_s1", "k_flux_s2"}, {"k_flux_tau0_s1", "k_flux_tau0_s2"}};
  const char* nm = BC == 0 ? names[tau0][stage - 1] : (BC == 1 ? "k_flux_wall" : "k_flux_farfield");
  if (tau0) {  // tau = 0: no non-equilibrium part, the Prandtl fix is identically zero (R29)
    if (stage == 1) launch(s, nm, [&] { L::template flux<NV, 1, true, BC, DQ0, false>(nb, s->stream, a); });
    else launch(s, nm, [&] { L::template flux<NV, 2, true, BC, DQ0, false>(nb, s->stream, a); });
  } else {
    if (stage == 1) launch(s, nm, [&] { L::template flux<NV, 1, false, BC, DQ0, PR>(nb, s->stream, a); });
    else launch(s, nm, [&] { L::template flux<NV, 2, false, BC, DQ0, PR>(nb, s->stream, a); });
  }
}

// dq0 readings other than R9 and the Prandtl fix exist for the fp64 path only (hgks_init
// rejects them for fp32); the Prandtl fix is built with the R9 reading
template <class L, int NV, int BC>
void launch_flux(hgks_solver* s, const typename L::FluxArgsT& a, int stage, bool tau0) {
  if constexpr (sizeof(typename L::RealT) == 8) {
    if (s->cfg.dq0_mode == 1) return launch_flux_q<L, NV, BC, 1>(s, a, stage, tau0);
    if (s->cfg.dq0_mode == 2) return launch_flux_q<L, NV, BC, 2>(s, a, stage, tau0);
    if (s->gp.pr_fac != 0.0) return launch_flux_q<L, NV, BC, 0, true>(s, a, stage, tau0);
  }
  launch_flux_q<L, NV, BC, 0>(s, a, stage, tau0);
}

// the faces of one kind (NV vertices)
template <class L, int NV>
void run_flux_nv(hgks_solver* s, typename L::FluxArgsT a, int stage, int part) {
  const FaceClass& F = s->rp->fcls[NV == 3 ? 0 : 1];
  const bool tau0 = s->cfg.tau_mode == 0;
  // part 0: early interior faces; 1: late interior + wall + farfield; 2: all
  const int64_t b = F.base;
  const int64_t i0 = part == 1 ? F.n_if_early : 0, i1 = part == 0 ? F.n_if_early : F.n_if;
  const int64_t ranges[3][2] = {{b + i0, i1 - i0},
                                {b + F.n_if, part == 0 ? 0 : F.n_wf},
                                {b + F.n_if + F.n_wf, part == 0 ? 0 : F.n_ff}};
  for (int bc = 0; bc < 3; ++bc) {
    a.face0 = (int)ranges[bc][0];
    a.n_faces = (int)ranges[bc][1];
    if (a.n_faces == 0) continue;
    if (bc == 0) launch_flux<L, NV, 0>(s, a, stage, tau0);
    else if (bc == 1) launch_flux<L, NV, 1>(s, a, stage, tau0);
    else launch_flux<L, NV, 2>(s, a, stage, tau0);
  }
}

template <class L>
void run_flux(hgks_solver* s, const void* Q, int stage, int part) {
  const RankPlan& rp = *s->rp;
  typename L::FluxArgsT a;
  a.Q = as<L>(Q);
  a.ceff = as<L>(s->d.ceff);
  a.ceff0 = s->d.ceff0 ? as<L>(s->d.ceff0) : nullptr;
  a.f_cells = s->d.f_cells;
  a.f_geo = as<L>(s->d.f_geo);
  a.f_stride = rp.f_geo_stride;
  a.n_faces = 0;
  a.face0 = 0;
  a.F1 = as<L>(s->d.F1);
  a.F2 = as<L>(s->d.F2);
  a.ctrl = s->d.ctrl;
  a.gp = make_gas_for<L>(s->gp);
  // triangles (tets, prism ends), then quadrilaterals (hexes, prism sides)
  if (s->lay.cell_type != 8) run_flux_nv<L, 3>(s, a, stage, part);
  if (s->lay.cell_type != 4) run_flux_nv<L, 4>(s, a, stage, part);
}

template <class L>
typename L::UpdateArgsT update_args(hgks_solver* s) {
  typename L::UpdateArgsT u;
  u.Q = as<L>(s->d.Q);
  u.R = as<L>(s->d.R);
  u.F1 = as<L>(s->d.F1);
  u.F2 = as<L>(s->d.F2);
  u.cf = s->d.cf;
  u.inv_v = as<L>(s->d.inv_v);
  u.h_dt = as<L>(s->d.h_dt);
  u.n_owned = (int)s->rp->n_owned;
  u.ctrl = s->d.ctrl;
  u.gp = s->gp;
  return u;
}

template <class L>
void pack(hgks_solver* s, const void* Q) {
  const int ns = (int)s->rp->send_list.size();
  if (ns > 0)
    launch(s, "k_pack",
           [&] { L::pack(blocks(3 * ns, 256), s->stream, as<L>(Q), s->d.send_list, ns, as<L>(s->d.sendbuf)); });
}

// a5: halo exchange of the 3 ghost layers.  NCCL transport: grouped
// send/recv per peer straight into the contiguous ghost ranges (no unpack).
// Loopback transport: done by hgks_group_step across the solvers of one process.
template <class L>
void exchange(hgks_solver* s, void* Q) {
  const RankPlan& rp = *s->rp;
  if (s->n_ranks == 1 || rp.peers.empty() || s->transport != HGKS_TRANSPORT_NCCL) return;
  pack<L>(s, Q);
  CUDA_TRY(cudaEventRecord(s->ev_packed, s->stream));
  CUDA_TRY(cudaStreamWaitEvent(s->comm_stream, s->ev_packed, 0));
  const int dtype = s->fp32 ? ncclFloat32 : ncclFloat64;
  typename L::RealT* q = as<L>(Q);
  typename L::RealT* sb = as<L>(s->d.sendbuf);
  Nccl& N = nccl();
  NCCL_TRY(N.GroupStart());
  for (size_t p = 0; p < rp.peers.size(); ++p) {
    if (rp.send_cnt[p] > 0)
      NCCL_TRY(N.Send(sb + (size_t)QS * rp.send_off[p], (size_t)QS * rp.send_cnt[p], dtype, rp.peers[p], s->comm,
                      s->comm_stream));
    if (rp.recv_cnt[p] > 0)
      NCCL_TRY(N.Recv(q + (size_t)QS * rp.recv_off[p], (size_t)QS * rp.recv_cnt[p], dtype, rp.peers[p], s->comm,
                      s->comm_stream));
  }
  NCCL_TRY(N.GroupEnd());
  CUDA_TRY(cudaEventRecord(s->ev_halo, s->comm_stream));
}

// f3: fused halo put for the loopback group -- one k_put per sending rank writes its send
// rows straight into the receivers' ghost rows (replaces k_pack + one device copy per
// peer pair).  The (receiver, row) map comes from the two ranks' plans (recv_off of the
// receiver's range for this sender + position in the sender's range for that peer).
// What a sender needs to know about a receiver: where the receiver keeps the ghost rows
// each of its peers sends (its recv_off / recv_cnt per peer).
struct RecvTab {
  int32_t n = 0;
  int32_t peer[kMaxGroup];
  int64_t off[kMaxGroup], cnt[kMaxGroup];
};
RecvTab recv_tab(const RankPlan& rp) {
  RecvTab t;
  if (rp.peers.size() > (size_t)kMaxGroup) throw Error(HGKS_E_ARG, "more than 16 exchange peers");
  for (size_t k = 0; k < rp.peers.size(); ++k) {
    t.peer[t.n] = rp.peers[k];
    t.off[t.n] = rp.recv_off[k];
    t.cnt[t.n++] = rp.recv_cnt[k];
  }
  return t;
}

// (receiver rank, receiver row) of every send row of rank q: the k-th row q sends to p lands
// at p's recv_off for q plus k (both sides order these cells by global id)
template <class TabOf>
std::vector<int2> put_map(const RankPlan& rq, int q, TabOf&& tab_of) {
  std::vector<int2> dst(rq.send_list.size(), int2{-1, -1});
  for (size_t ip = 0; ip < rq.peers.size(); ++ip) {
    if (rq.send_cnt[ip] == 0) continue;
    const int p = rq.peers[ip];
    const RecvTab& tp = tab_of(p);
    int iq = 0;
    while (iq < tp.n && tp.peer[iq] != q) ++iq;
    if (iq == tp.n || tp.cnt[iq] != rq.send_cnt[ip])
      throw Error(HGKS_E_STATE, "inconsistent exchange plans between ranks");
    for (int64_t k = 0; k < rq.send_cnt[ip]; ++k) dst[rq.send_off[ip] + k] = int2{p, (int)(tp.off[iq] + k)};
  }
  return dst;
}

// the put map of rank q from the plans of one mesh object (whole-mesh builds)
std::vector<int2> put_map_mesh(hgks_mesh* m, int q) {
  std::map<int, RecvTab> tabs;
  return put_map(m->plan(q), q, [&](int p) -> const RecvTab& {
    auto it = tabs.find(p);
    if (it == tabs.end()) it = tabs.emplace(p, recv_tab(m->plan(p))).first;
    return it->second;
  });
}

// loopback group: each solver's own plan (its mesh may be a region build)
void build_put_map(hgks_solver* const* ss, int n) {
  std::vector<RecvTab> tabs(n);
  for (int p = 0; p < n; ++p) tabs[p] = recv_tab(*ss[p]->rp);
  for (int q = 0; q < n; ++q) {
    hgks_solver* s = ss[q];
    if (s->put_ready) continue;
    std::vector<int2> dst = put_map(*s->rp, q, [&](int p) -> const RecvTab& { return tabs[p]; });
    if (!dst.empty())
      CUDA_TRY(cudaMemcpy(s->d.put_dst, dst.data(), dst.size() * sizeof(int2), cudaMemcpyHostToDevice));
    s->put_ready = true;
  }
}

template <class L>
void put(hgks_solver* const* ss, int q, int n) {
  hgks_solver* s = ss[q];
  const int ns = (int)s->rp->send_list.size();
  if (ns == 0) return;
  typename L::PeerQT peer{};
  for (int k = 0; k < n; ++k) peer.q[k] = as<L>(ss[k]->d.Q);
  launch(s, "k_put", [&] {
    L::put(blocks(3 * ns, 256), s->stream, as<L>(s->d.Q), s->d.send_list, s->d.put_dst, ns, peer);
  });
}

// the compute stream waits for the ghosts (no-op without an NCCL exchange in flight)
void wait_halo(hgks_solver* s) {
  if (s->n_ranks == 1 || s->rp->peers.empty() || s->transport != HGKS_TRANSPORT_NCCL) return;
  CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_halo, 0));
}

// a4: global min of the CFL bound (exact, order independent).  Enqueued on the comm stream
// after the work that produced the local bound; the compute stream waits for it only in
// begin_step (or before anything reads or resets the bound), so it overlaps the next step's
// stage-1 reconstruction and flux.
void allreduce_dt(hgks_solver* s) {
  if (s->n_ranks == 1 || s->transport == HGKS_TRANSPORT_LOOPBACK) return;
  CUDA_TRY(cudaEventRecord(s->ev_upd2, s->stream));
  CUDA_TRY(cudaStreamWaitEvent(s->comm_stream, s->ev_upd2, 0));
  NCCL_TRY(nccl().AllReduce(&s->d.ctrl->dtmin_bits, &s->d.ctrl->dtmin_bits, 1, ncclUint64, ncclMin, s->comm,
                            s->comm_stream));
  CUDA_TRY(cudaEventRecord(s->ev_dt, s->comm_stream));
  s->dt_pending = true;
}

// the compute stream waits for the last min(dt) allreduce (no-op if none is in flight)
void wait_dt(hgks_solver* s) {
  if (!s->dt_pending) return;
  CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_dt, 0));
  s->dt_pending = false;
}

// this step's time bookkeeping (dt from the global min, t_stop clipping); deferred on
// multi-rank solvers to the first point of stage 1 that needs dt
void begin_step(hgks_solver* s) {
  if (!s->begin_pending) return;
  wait_dt(s);
  launch(s, "k_step_begin",
         [&] { k_step_begin<<<1, 1, 0, s->stream>>>(s->d.ctrl, s->cfg.cfl, s->cfg.fixed_dt, s->cur_t_stop); });
  s->begin_pending = false;
}

template <class L>
void bc_ghosts(hgks_solver* s, void* Q, int part) {
  const RankPlan& rp = *s->rp;
  if (rp.n_bghost == 0) return;
  const int first = (int)(rp.n_owned + rp.n_pghost);
  launch(s, "k_bc_ghosts", [&] {
    L::bc_ghosts(blocks(rp.n_bghost, 128), s->stream, as<L>(Q), first, (int)rp.n_bghost, s->d.bg_cell, s->d.bg_bc,
                 as<L>(s->d.bg_normal), make_gas_for<L>(s->gp), (int)rp.n_owned, part);
  });
}

// work of one stage that needs no partition-ghost data (overlaps the exchange)
template <class L>
void stage_early(hgks_solver* s, int st) {
  bc_ghosts<L>(s, s->d.Q, 0);
  run_recon<L>(s, s->d.Q, 0);
  if (s->cfg.tau_mode != 0) begin_step(s);  // the NS collision time needs dt (R7)
  run_flux<L>(s, s->d.Q, st, 0);
}

// the rest of the stage, after the ghosts are current
template <class L>
void stage_late(hgks_solver* s, int st) {
  bc_ghosts<L>(s, s->d.Q, 1);
  run_recon<L>(s, s->d.Q, 1);
  run_flux<L>(s, s->d.Q, st, 1);
  begin_step(s);  // tau = 0: dt is first needed by the stage-1 update
  const typename L::UpdateArgsT u = update_args<L>(s);
  const int n = (int)s->rp->n_owned;
  const int nf = s->lay.nfaces;
  if (st == 1) {
    if (nf == 4) launch(s, "k_update1", [&] { L::template update1<4>(blocks(n, 256), s->stream, u); });
    else if (nf == 5) launch(s, "k_update1", [&] { L::template update1<5>(blocks(n, 256), s->stream, u); });
    else launch(s, "k_update1", [&] { L::template update1<6>(blocks(n, 256), s->stream, u); });
  } else {
    if (nf == 4) launch(s, "k_update2", [&] { L::template update2<4>(blocks(n, 256), s->stream, u); });
    else if (nf == 5) launch(s, "k_update2", [&] { L::template update2<5>(blocks(n, 256), s->stream, u); });
    else launch(s, "k_update2", [&] { L::template update2<6>(blocks(n, 256), s->stream, u); });
  }
}

// f3 across processes (HGKS_TRANSPORT_P2P): the owner puts its send rows straight into
// the receivers' ghost rows over NVLink (peer memory mapped by CUDA IPC), ordered by
// per-stage epoch flags: (1) wait until every receiver has finished reading the ghost
// rows of the previous stage, (2)+(3) k_put_release: the puts, a system-scope fence by every
// thread and, from the last block, the release of "stage e arrived" to the receivers,
// (4) ghost-free work, (5) acquire "arrived" from every sender, (6) the rest of the
// stage, (7) release "stage e consumed" to the senders.  Graph capture is off for
// n_ranks > 1, so the host-side epoch values are baked into eager launches.
template <class L>
void stage_p2p(hgks_solver* s, int st) {
  const unsigned long long e = ++s->epoch;
  P2PWait w_cons{}, w_arr{};
  P2PSignal s_arr{}, s_cons{};
  for (int p : s->put_to) {
    w_cons.src[w_cons.n++] = &s->d.flags->consumed[p];
    s_arr.dst[s_arr.n++] = &s->peer_flags[p]->arrived[s->rank];
  }
  for (int q : s->recv_from) {
    w_arr.src[w_arr.n++] = &s->d.flags->arrived[q];
    s_cons.dst[s_cons.n++] = &s->peer_flags[q]->consumed[s->rank];
  }
  if (e > 1 && w_cons.n) launch(s, "k_p2p_wait", [&] { k_p2p_wait<<<1, 32, 0, s->stream>>>(w_cons, e - 1); });
  const int ns = (int)s->rp->send_list.size();
  if (ns) {  // put + system-scope release of "stage e arrived" in one kernel (k_put_release)
    typename L::PeerQT peer{};
    for (int p : s->put_to) peer.q[p] = as<L>(s->peer_Q[p]);
    launch(s, "k_put_release", [&] {
      L::put_release(blocks(3 * ns, 256), s->stream, as<L>(s->d.Q), s->d.send_list, s->d.put_dst, ns, peer, s_arr, e,
                     &s->d.flags->put_blocks);
    });
  } else if (s_arr.n) {
    launch(s, "k_p2p_signal", [&] { k_p2p_signal<<<1, 32, 0, s->stream>>>(s_arr, e); });
  }
  stage_early<L>(s, st);
  if (w_arr.n) launch(s, "k_p2p_wait", [&] { k_p2p_wait<<<1, 32, 0, s->stream>>>(w_arr, e); });
  stage_late<L>(s, st);
  if (s_cons.n) launch(s, "k_p2p_signal", [&] { k_p2p_signal<<<1, 32, 0, s->stream>>>(s_cons, e); });
  if (st == 2) allreduce_dt(s);
}

template <class L>
void stage(hgks_solver* s, int st) {
  if (s->transport == HGKS_TRANSPORT_P2P && s->n_ranks > 1) return stage_p2p<L>(s, st);
  exchange<L>(s, s->d.Q);  // NCCL on the comm stream
  stage_early<L>(s, st);
  wait_halo(s);
  stage_late<L>(s, st);
  if (st == 2) allreduce_dt(s);
}

template <class L>
void init_dt(hgks_solver* s) {
  const int n = (int)s->rp->n_owned;
  launch(s, "k_dt_init",
         [&] { L::dt_init(blocks(n, 256), s->stream, as<L>(s->d.Q), as<L>(s->d.h_dt), n, s->d.ctrl, s->gp); });
  allreduce_dt(s);
}

// asynchronous on the stream: H2D of the caller's rows, scatter into the local
// rows, reset time, recompute the CFL bound
template <class L>
void upload_state(hgks_solver* s, const double* h_Q, double t) {
  wait_dt(s);  // k_reset_ctrl rewrites the bound an allreduce may still be reducing
  const RankPlan& rp = *s->rp;
  const int n = (int)rp.n_owned;
  const int k = s->in_slot;
  s->in_slot ^= 1;
  // the H2D into slot k waits until the scatter that last read slot k is done
  CUDA_TRY(cudaStreamWaitEvent(s->h2d_stream, s->ev_scattered[k], 0));
  if (s->n_ranks == 1) {
    CUDA_TRY(cudaMemcpyAsync(s->d.stage_in[k], h_Q, sizeof(double) * 5 * s->mesh->gm.nc, cudaMemcpyHostToDevice,
                             s->h2d_stream));
  } else {
    // gather this rank's rows into pinned staging slot k (its previous copy must be done)
    CUDA_TRY(cudaEventSynchronize(s->ev_h2d[k]));
    double* hs = s->pinned[k];
    for (int i = 0; i < n; ++i) std::memcpy(hs + 5 * (size_t)i, h_Q + 5 * rp.l2g[i], 5 * sizeof(double));
    CUDA_TRY(cudaMemcpyAsync(s->d.stage_in[k], hs, sizeof(double) * 5 * n, cudaMemcpyHostToDevice, s->h2d_stream));
  }
  CUDA_TRY(cudaEventRecord(s->ev_h2d[k], s->h2d_stream));
  CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_h2d[k], 0));
  launch(s, "k_scatter_state",
         [&] { L::scatter(blocks(n, 256), s->stream, s->d.stage_in[k], s->d.in_row, n, as<L>(s->d.Q)); });
  CUDA_TRY(cudaEventRecord(s->ev_scattered[k], s->stream));
  launch(s, "k_reset_ctrl", [&] { k_reset_ctrl<<<1, 1, 0, s->stream>>>(s->d.ctrl, t); });
  init_dt<L>(s);
}

// enqueue: gather the owned rows (ascending global id) into staging slot k on the
// compute stream, then the D2H into h_Q on the copy stream
void download_state(hgks_solver* s, double* h_Q) {
  const int n = (int)s->rp->n_owned;
  const int k = s->out_slot;
  s->out_slot ^= 1;
  CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_d2h[k], 0));  // slot k's previous D2H is done
  launch(s, "k_gather_state", [&] {
    if (s->fp32)
      p32::Launch::gather(blocks(n, 256), s->stream, (const float*)s->d.Q, s->d.out_local, n, s->d.stage_out[k]);
    else
      p64::Launch::gather(blocks(n, 256), s->stream, (const double*)s->d.Q, s->d.out_local, n, s->d.stage_out[k]);
  });
  CUDA_TRY(cudaEventRecord(s->ev_gathered[k], s->stream));
  CUDA_TRY(cudaStreamWaitEvent(s->d2h_stream, s->ev_gathered[k], 0));
  CUDA_TRY(cudaMemcpyAsync(h_Q, s->d.stage_out[k], sizeof(double) * 5 * n, cudaMemcpyDeviceToHost, s->d2h_stream));
  CUDA_TRY(cudaEventRecord(s->ev_d2h[k], s->d2h_stream));
}

// the compute stream waits for every enqueued copy; then the host waits for it
void sync_all(hgks_solver* s) {
  for (int k = 0; k < 2; ++k) {
    CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_h2d[k], 0));
    CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_d2h[k], 0));
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
}

// precision dispatch of the hot path
#define HGKS_DISPATCH(s, fn, ...) \
  ((s)->fp32 ? fn<p32::Launch>(__VA_ARGS__) : fn<p64::Launch>(__VA_ARGS__))

}  // namespace

// ============================================================================
// C-ABI
// ============================================================================
extern "C" {

const char* hgks_last_error(void) { return g_last_error.c_str(); }
const char* hgks_version(void) { return "hgks-b200 0.1 (sm_100a, fp64)"; }

hgks_status hgks_mesh_create(const hgks_mesh_desc* d, hgks_mesh** out) {
  return guard([&] {
    if (!d || !out) throw Error(HGKS_E_ARG, "null argument");
    auto m = std::make_unique<hgks_mesh>();
    m->gm = build_global_mesh(d->xyz, d->n_nodes, d->cell_type, d->cell_nodes, d->n_cells, d->periodic_origin,
                              d->periodic_length, d->bface_nodes, d->bface_tag, d->n_bfaces, d->n_ranks, d->cell_part,
                              d->rank_only);
    *out = m.release();
  });
}

hgks_status hgks_mesh_destroy(hgks_mesh* m) {
  delete m;
  return HGKS_OK;
}

hgks_status hgks_mesh_info(const hgks_mesh* mc, int32_t rank, hgks_mesh_stats* st) {
  return guard([&] {
    if (!mc || !st) throw Error(HGKS_E_ARG, "null argument");
    hgks_mesh* m = const_cast<hgks_mesh*>(mc);
    const RankPlan& rp = m->plan(rank);
    std::memset(st, 0, sizeof(*st));
    st->n_cells_global = m->gm.nc_global;
    st->n_owned = rp.n_owned;
    st->n_ghost = rp.n_pghost;
    for (int k = 0; k < 3; ++k) st->ghost_layer[k] = rp.ghost_layer[k];
    st->n_bghost = rp.n_bghost;
    st->n_faces = rp.n_faces;
    st->n_faces_bc = rp.n_wf + rp.n_ff;
    st->stencil_min = rp.stencil_min;
    st->stencil_max = rp.stencil_max;
    st->n_sub = m->gm.lay.M;
    st->n_peers = (int32_t)rp.peers.size();
    st->send_cells = (int64_t)rp.send_list.size();
    for (auto c : rp.recv_cnt) st->recv_cells += c;
    st->edge_cut = m->gm.edge_cut;
    st->edge_cut_rcb = m->gm.edge_cut_rcb ? m->gm.edge_cut_rcb : m->gm.edge_cut;
    st->rank_cut_faces = rp.rank_cut_faces;
    st->n_early_cells = rp.n_recon_early;
    st->n_early_faces = rp.n_if_early;
  });
}

hgks_status hgks_workspace_size(const hgks_mesh* mc, const hgks_config* cfg, int32_t rank, size_t* bytes) {
  return guard([&] {
    if (!mc || !bytes) throw Error(HGKS_E_ARG, "null argument");
    (void)cfg;
    hgks_mesh* m = const_cast<hgks_mesh*>(mc);
    const RankPlan& rp = m->plan(rank);
    Carve c{nullptr, 0, 0};
    DevArrays d;
    const bool fp32 = cfg && cfg->precision == 32;
    *bytes = layout(m->gm, rp, fp32 ? sizeof(float) : sizeof(double), cfg ? cfg->dq0_mode : 0, c, d);
  });
}

hgks_status hgks_init(const hgks_mesh* mc, const hgks_config* cfg, const hgks_dist* dist, void* d_ws, size_t ws_bytes,
                      void* stream, const double* h_Q0, hgks_solver** out) {
  return guard([&] {
    if (!mc || !cfg || !d_ws || !h_Q0 || !out) throw Error(HGKS_E_ARG, "null argument");
    hgks_mesh* m = const_cast<hgks_mesh*>(mc);
    auto s = std::make_unique<hgks_solver>();
    s->mesh = m;
    s->cfg = *cfg;
    s->rank = dist ? dist->rank : 0;
    s->n_ranks = dist ? dist->n_ranks : 1;
    s->transport = dist ? dist->transport : HGKS_TRANSPORT_NCCL;
    if (s->transport < HGKS_TRANSPORT_NCCL || s->transport > HGKS_TRANSPORT_P2P)
      throw Error(HGKS_E_ARG, "unknown transport");
    if (s->transport == HGKS_TRANSPORT_P2P && s->n_ranks > kMaxGroup)
      throw Error(HGKS_E_ARG, "HGKS_TRANSPORT_P2P supports at most 16 ranks (one node)");
    if (s->n_ranks != m->gm.n_ranks)
      throw Error(HGKS_E_ARG, "dist->n_ranks differs from the mesh partition (" + std::to_string(m->gm.n_ranks) + ")");
    if (dist) CUDA_TRY(cudaSetDevice(dist->device));
    CUDA_TRY(cudaGetDevice(&s->device));
    if (const char* e = std::getenv("HGKS_GRAPHS")) s->use_graphs = std::atoi(e) != 0;
    if (const char* e = std::getenv("HGKS_RECON_PAIR")) s->recon_pair = std::atoi(e) != 0 ? 1 : 0;
    s->stream = (cudaStream_t)stream;
    s->rp = &m->plan(s->rank);
    s->lay = m->gm.lay;
    const RankPlan& rp = *s->rp;
    if (cfg->gamma <= 1.0 || cfg->gamma > 5.0 / 3.0) throw Error(HGKS_E_ARG, "gamma out of range");
    if (!(cfg->cfl > 0) && !(cfg->fixed_dt > 0)) throw Error(HGKS_E_ARG, "need cfl > 0 or fixed_dt > 0");
    GasParams& g = s->gp;
    g.gamma = cfg->gamma;
    g.K = (5.0 - 3.0 * cfg->gamma) / (cfg->gamma - 1.0);
    g.cfl = cfg->cfl;
    g.fixed_dt = cfg->fixed_dt;
    g.eps = cfg->eps;
    g.omega_pow = cfg->omega_pow;
    g.tau_mode = cfg->tau_mode;
    g.c1 = cfg->c1;
    g.mu_inf = cfg->mu_inf;
    g.t_inf = cfg->t_inf;
    g.mu_exp = cfg->mu_exp;
    for (int k = 0; k < 5; ++k) g.fs[k] = cfg->freestream[k];
    if (cfg->prandtl < 0) throw Error(HGKS_E_ARG, "prandtl must be > 0 (0 = no correction)");
    g.pr_fac = (cfg->prandtl > 0 && cfg->prandtl != 1.0) ? 1.0 / cfg->prandtl - 1.0 : 0.0;
    if (cfg->precision != 64 && cfg->precision != 32) throw Error(HGKS_E_ARG, "precision must be 64 or 32");
    if (cfg->dq0_mode < 0 || cfg->dq0_mode > 2) throw Error(HGKS_E_ARG, "dq0_mode must be 0, 1 or 2");
    if (cfg->dq0_mode != 0 && cfg->precision == 32)
      throw Error(HGKS_E_ARG, "dq0_mode 1/2 (readings R9k/R9s) are built for the fp64 path only");
    if (g.pr_fac != 0.0 && (cfg->precision == 32 || cfg->dq0_mode != 0))
      throw Error(HGKS_E_ARG, "the Prandtl fix (R29) is built for the fp64 path with dq0_mode 0");
    s->fp32 = cfg->precision == 32;
    s->rs = s->fp32 ? sizeof(float) : sizeof(double);
    s->nq = (size_t)QS * round32(rp.n_local());
    Carve c{(char*)d_ws, 0, ws_bytes};
    if ((reinterpret_cast<uintptr_t>(d_ws) & 255) != 0) throw Error(HGKS_E_ARG, "workspace must be 256-byte aligned");
    layout(m->gm, rp, s->rs, cfg->dq0_mode, c, s->d);
    cudaStream_t st = s->stream;
    auto up = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    };
    // working-precision arrays: converted on the host for fp32 (kept alive until the sync below)
    std::vector<std::vector<float>> keep;
    auto upr = [&](void* dst, const std::vector<double>& v) {
      if (!s->fp32) return up(dst, v.data(), v.size() * sizeof(double));
      keep.emplace_back(v.begin(), v.end());
      up(dst, keep.back().data(), v.size() * sizeof(float));
    };
    up(s->d.recon_cell, rp.recon_cell.data(), rp.recon_cell.size() * sizeof(int));
    up(s->d.st_id, rp.st_id_tiled.data(), rp.st_id_tiled.size() * sizeof(int));

    up(s->d.sub_slot, rp.sub_slot.data(), rp.sub_slot.size());
    if (s->d.n_sub) up(s->d.n_sub, rp.n_sub.data(), rp.n_sub.size());
    upr(s->d.op, rp.op);
    upr(s->d.geo, rp.geo);
    up(s->d.st_shift, rp.st_shift.data(), rp.st_shift.size());
    upr(s->d.cgeo, rp.cgeo);
    up(s->d.f_cells, rp.f_cells.data(), rp.f_cells.size() * sizeof(int));
    upr(s->d.f_geo, rp.f_geo);
    up(s->d.cf, rp.cf.data(), rp.cf.size() * sizeof(int));
    upr(s->d.inv_v, rp.inv_v);
    upr(s->d.h_dt, rp.h_dt);
    up(s->d.bg_cell, rp.bg_cell.data(), rp.bg_cell.size() * sizeof(int));
    up(s->d.bg_bc, rp.bg_bc.data(), rp.bg_bc.size() * sizeof(int));
    upr(s->d.bg_normal, rp.bg_normal);
    up(s->d.send_list, rp.send_list.data(), rp.send_list.size() * sizeof(int));
    // state maps: in_row[i] = row of owned cell i in the caller's array (single
    // rank) or its position in the gathered staging array; out_local[k] = local
    // id of the k-th owned cell in ascending global id
    std::vector<int64_t> in_row(rp.n_owned);
    for (int64_t i = 0; i < rp.n_owned; ++i) in_row[i] = s->n_ranks == 1 ? rp.l2g[i] : i;
    std::vector<int> out_local(rp.n_owned);
    std::iota(out_local.begin(), out_local.end(), 0);
    std::sort(out_local.begin(), out_local.end(), [&](int a, int b) { return rp.l2g[a] < rp.l2g[b]; });
    up(s->d.in_row, in_row.data(), in_row.size() * sizeof(int64_t));
    up(s->d.out_local, out_local.data(), out_local.size() * sizeof(int));
    CUDA_TRY(cudaMemsetAsync(s->d.Q, 0, s->rs * s->nq, st));
    CUDA_TRY(cudaMemsetAsync((char*)s->d.F1 + s->rs * 10 * rp.n_faces, 0, s->rs * 10, st));
    CUDA_TRY(cudaMemsetAsync((char*)s->d.F2 + s->rs * 5 * rp.n_faces, 0, s->rs * 5, st));
    CUDA_TRY(cudaMemsetAsync(s->d.flags, 0, sizeof(P2PFlags), st));
    Ctrl h{};
    h.bad_cell = INT_MAX;
    h.dtmin_bits = 0x7fefffffffffffffull;
    up(s->d.ctrl, &h, sizeof(Ctrl));
    if (s->n_ranks > 1 && s->transport != HGKS_TRANSPORT_LOOPBACK) {
      Nccl& N = nccl();
      if (!N.h || !N.CommInitRank) throw Error(HGKS_E_NCCL, "libnccl.so.2 not found");
      ncclUniqueId id;
      std::memcpy(id.internal, dist->nccl_id, 128);
      NCCL_TRY(N.CommInitRank(&s->comm, s->n_ranks, id, s->rank));
      CUDA_TRY(cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&s->ev_packed, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&s->ev_halo, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&s->ev_upd2, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&s->ev_dt, cudaEventDisableTiming));
    }
    if (s->n_ranks > 1)
      for (int k = 0; k < 2; ++k)
        CUDA_TRY(cudaMallocHost(&s->pinned[k], sizeof(double) * 5 * std::max<int64_t>(1, rp.n_owned)));
    CUDA_TRY(cudaStreamCreateWithFlags(&s->h2d_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&s->d2h_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      for (cudaEvent_t* e : {&s->ev_h2d[k], &s->ev_scattered[k], &s->ev_gathered[k], &s->ev_d2h[k]}) {
        CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(*e, st));  // "already complete" for the first waits
      }
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    HGKS_DISPATCH(s, upload_state, s.get(), h_Q0, 0.0);
    CUDA_TRY(cudaStreamSynchronize(st));
    *out = s.release();
  });
}

hgks_status hgks_destroy(hgks_solver* s) {
  return guard([&] {
    if (!s) return;
    cudaStreamSynchronize(s->stream);
    for (auto& kv : s->kstat)
      for (auto& e : kv.second.pending) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
    for (auto e : s->event_pool) cudaEventDestroy(e);
    for (int k = 0; k < kMaxGroup; ++k)
      if (s->peer_base[k]) cudaIpcCloseMemHandle(s->peer_base[k]);
    if (s->comm_stream) cudaStreamSynchronize(s->comm_stream);  // a min(dt) allreduce may be in flight
    if (s->comm && nccl().CommDestroy) nccl().CommDestroy(s->comm);
    if (s->comm_stream) cudaStreamDestroy(s->comm_stream);
    if (s->ev_packed) cudaEventDestroy(s->ev_packed);
    if (s->ev_halo) cudaEventDestroy(s->ev_halo);
    if (s->ev_upd2) cudaEventDestroy(s->ev_upd2);
    if (s->ev_dt) cudaEventDestroy(s->ev_dt);
    cudaStreamSynchronize(s->h2d_stream);
    cudaStreamSynchronize(s->d2h_stream);
    for (int k = 0; k < 2; ++k) {
      if (s->pinned[k]) cudaFreeHost(s->pinned[k]);
      for (cudaEvent_t e : {s->ev_h2d[k], s->ev_scattered[k], s->ev_gathered[k], s->ev_d2h[k]})
        if (e) cudaEventDestroy(e);
    }
    if (s->h2d_stream) cudaStreamDestroy(s->h2d_stream);
    if (s->step_graph) cudaGraphExecDestroy(s->step_graph);
    if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
    if (s->d2h_stream) cudaStreamDestroy(s->d2h_stream);
    delete s;
  });
}

hgks_status hgks_step(hgks_solver* s, int32_t n_steps, double t_stop, hgks_step_info* info) {
  return guard([&] {
    if (!s || n_steps < 0) throw Error(HGKS_E_ARG, "bad argument");
    if (s->transport == HGKS_TRANSPORT_P2P && s->n_ranks > 1 && !s->p2p_ready)
      throw Error(HGKS_E_STATE, "HGKS_TRANSPORT_P2P: call hgks_p2p_connect on every rank first");
    if (s->transport == HGKS_TRANSPORT_LOOPBACK && s->n_ranks > 1 && n_steps > 0)
      throw Error(HGKS_E_STATE,
                  "HGKS_TRANSPORT_LOOPBACK solver of a multi-rank group: advance the group with hgks_group_step "
                  "(hgks_step would run without a halo exchange or a global dt)");
    Ctrl before{};
    if (info) {
      CUDA_TRY(cudaMemcpyAsync(&before, s->d.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s->stream));
      CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    auto one_step = [&] {
      s->begin_pending = true;
      s->cur_t_stop = t_stop;
      // one rank: begin at once (graph replays); several: where stage 1 first needs dt
      if (s->n_ranks == 1 || s->transport == HGKS_TRANSPORT_LOOPBACK) begin_step(s);
      HGKS_DISPATCH(s, stage, s, 1);
      HGKS_DISPATCH(s, stage, s, 2);
    };
    // graphs: single rank, not profiling, after one eager step (one-time attribute setup)
    const bool graphs = s->use_graphs && s->n_ranks == 1 && !s->profiling && s->eager_steps > 0;
    if (graphs && (!s->step_graph || s->graph_t_stop != t_stop)) {
      if (s->step_graph) CUDA_TRY(cudaGraphExecDestroy(s->step_graph));
      s->step_graph = nullptr;
      if (!s->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
      cudaStream_t user = s->stream;
      const int64_t l0 = s->launches;
      cudaGraph_t g = nullptr;
      s->stream = s->cap_stream;
      CUDA_TRY(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      try {
        one_step();
      } catch (...) {
        cudaStreamEndCapture(s->stream, &g);
        if (g) cudaGraphDestroy(g);
        s->stream = user;
        throw;
      }
      CUDA_TRY(cudaStreamEndCapture(s->stream, &g));
      s->stream = user;
      CUDA_TRY(cudaGraphInstantiate(&s->step_graph, g, 0));
      CUDA_TRY(cudaGraphDestroy(g));
      s->graph_launches = s->launches - l0;
      s->launches = l0;
      s->graph_t_stop = t_stop;
    }
    for (int k = 0; k < n_steps; ++k) {
      if (graphs) {
        CUDA_TRY(cudaGraphLaunch(s->step_graph, s->stream));
        s->launches += s->graph_launches;
      } else {
        one_step();
        ++s->eager_steps;
      }
    }
    if (info) {
      wait_dt(s);
      Ctrl h;
      CUDA_TRY(cudaMemcpyAsync(&h, s->d.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s->stream));
      CUDA_TRY(cudaStreamSynchronize(s->stream));
      info->steps_done = h.steps - before.steps;
      info->t = h.t_next;
      info->last_dt = h.dt;
      info->fallbacks = h.fallbacks;
      if (h.bad_cell != INT_MAX) {
        int64_t gid = h.bad_cell < (int)s->rp->l2g.size() ? s->rp->l2g[h.bad_cell] : -1;
        throw Error(HGKS_E_POSITIVITY, "non-positive density or pressure at cell " + std::to_string(gid));
      }
      if (!(h.dt >= 0.0) || !std::isfinite(h.t_next)) throw Error(HGKS_E_STATE, "non-finite time step");
    }
  });
}

hgks_status hgks_set_state(hgks_solver* s, const double* h_Q, double t) {
  return guard([&] {
    if (!s || !h_Q) throw Error(HGKS_E_ARG, "null argument");
    HGKS_DISPATCH(s, upload_state, s, h_Q, t);
  });
}

hgks_status hgks_get_state(const hgks_solver* sc, double* h_Q, int64_t* h_gid, double* t) {
  return guard([&] {
    hgks_solver* s = const_cast<hgks_solver*>(sc);
    if (!s || !h_Q) throw Error(HGKS_E_ARG, "null argument");
    const int n = (int)s->rp->n_owned;
    download_state(s, h_Q);
    Ctrl h;
    CUDA_TRY(cudaMemcpyAsync(&h, s->d.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s->stream));
    sync_all(s);
    if (t) *t = h.t_next;
    if (h_gid) {
      std::vector<int64_t> g(s->rp->l2g.begin(), s->rp->l2g.begin() + n);
      std::sort(g.begin(), g.end());
      std::memcpy(h_gid, g.data(), sizeof(int64_t) * n);
    }
  });
}

hgks_status hgks_get_state_async(hgks_solver* s, double* h_Q) {
  return guard([&] {
    if (!s || !h_Q) throw Error(HGKS_E_ARG, "null argument");
    download_state(s, h_Q);
  });
}

hgks_status hgks_sync(hgks_solver* s) {
  return guard([&] {
    if (!s) throw Error(HGKS_E_ARG, "null solver");
    sync_all(s);
  });
}

hgks_status hgks_debug_residual(hgks_solver* s, const double* h_Q, double dt, double* h_L, double* h_dL) {
  return guard([&] {
    if (!s || !h_Q || !h_L || !h_dL) throw Error(HGKS_E_ARG, "null argument");
    if (s->n_ranks != 1) throw Error(HGKS_E_ARG, "hgks_debug_residual is single-rank only");
    const int n = (int)s->rp->n_owned;
    // save state, load h_Q, run stage-1 reconstruction + flux, restore
    CUDA_TRY(cudaMemcpyAsync(s->d.Qtmp, s->d.Q, s->rs * s->nq, cudaMemcpyDeviceToDevice, s->stream));
    Ctrl saved;
    CUDA_TRY(cudaMemcpyAsync(&saved, s->d.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    sync_all(s);  // no copy in flight may touch the staging slots
    CUDA_TRY(cudaMemcpyAsync(s->d.stage_in[0], h_Q, sizeof(double) * 5 * s->mesh->gm.nc, cudaMemcpyHostToDevice,
                             s->stream));
    launch(s, "k_scatter_state", [&] {
      if (s->fp32) p32::Launch::scatter(blocks(n, 256), s->stream, s->d.stage_in[0], s->d.in_row, n, (float*)s->d.Q);
      else p64::Launch::scatter(blocks(n, 256), s->stream, s->d.stage_in[0], s->d.in_row, n, (double*)s->d.Q);
    });
    Ctrl h = saved;
    h.dt = dt;
    CUDA_TRY(cudaMemcpyAsync(s->d.ctrl, &h, sizeof(Ctrl), cudaMemcpyHostToDevice, s->stream));
    HGKS_DISPATCH(s, bc_ghosts, s, s->d.Q, 2);
    HGKS_DISPATCH(s, run_recon, s, s->d.Q, 2);
    HGKS_DISPATCH(s, run_flux, s, s->d.Q, 1, 2);
    // L = (Q* - Q) ... computed directly on host from face fluxes for clarity
    std::vector<double> F1((size_t)10 * s->rp->n_faces);
    std::vector<int> cf(s->rp->cf);
    std::vector<float> F1f(s->fp32 ? F1.size() : 0);
    if (s->fp32)
      CUDA_TRY(cudaMemcpyAsync(F1f.data(), s->d.F1, F1f.size() * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
    else
      CUDA_TRY(cudaMemcpyAsync(F1.data(), s->d.F1, F1.size() * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->d.Q, s->d.Qtmp, s->rs * s->nq, cudaMemcpyDeviceToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->d.ctrl, &saved, sizeof(Ctrl), cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (s->fp32) std::copy(F1f.begin(), F1f.end(), F1.begin());
    const int NF = s->lay.nfaces;
    for (int i = 0; i < n; ++i) {
      double L[5] = {0, 0, 0, 0, 0}, dL[5] = {0, 0, 0, 0, 0};
      for (int p = 0; p < NF; ++p) {
        int e = cf[(size_t)p * n + i];
        int f = e >= 0 ? e : ~e;
        if (f >= s->rp->n_faces) continue;  // no face p (hybrid meshes)
        double sg = e >= 0 ? -1.0 : 1.0;
        for (int v = 0; v < 5; ++v) {
          L[v] += sg * F1[(size_t)f * 10 + v];
          dL[v] += sg * F1[(size_t)f * 10 + 5 + v];
        }
      }
      int64_t gid = s->rp->l2g[i];
      for (int v = 0; v < 5; ++v) {
        h_L[gid * 5 + v] = L[v] * s->rp->inv_v[i];
        h_dL[gid * 5 + v] = dL[v] * s->rp->inv_v[i];
      }
    }
  });
}

hgks_status hgks_set_profiling(hgks_solver* s, int32_t enabled) {
  return guard([&] {
    if (!s) throw Error(HGKS_E_ARG, "null solver");
    s->profiling = enabled != 0;
  });
}

hgks_status hgks_kernel_times(hgks_solver* s, int32_t cap, char (*names)[32], int64_t* launches, double* total_ms,
                              int32_t* n) {
  return guard([&] {
    if (!s || !n) throw Error(HGKS_E_ARG, "null argument");
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    int k = 0;
    for (auto& kv : s->kstat) {
      KStat& st = kv.second;
      for (auto& e : st.pending) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
        st.ms += ms;
        s->event_pool.push_back(e.first);
        s->event_pool.push_back(e.second);
      }
      st.pending.clear();
      if (k < cap) {
        std::snprintf(names[k], 32, "%s", kv.first.c_str());
        launches[k] = st.timed;
        total_ms[k] = st.ms;
      }
      ++k;
    }
    *n = std::min(k, cap);
  });
}

hgks_status hgks_nccl_unique_id(uint8_t* out) {
  return guard([&] {
    if (!out) throw Error(HGKS_E_ARG, "null argument");
    Nccl& N = nccl();
    if (!N.h || !N.GetUniqueId) throw Error(HGKS_E_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    NCCL_TRY(N.GetUniqueId(&id));
    std::memcpy(out, id.internal, 128);
  });
}

// Mechanics of the P2P transport's kernels on one device, with no rank waiting on
// another: k_put through a pointer table (fp64 rows into a second buffer), k_p2p_signal
// publishing an epoch, the flag read back, then k_p2p_wait on a flag that already holds
// the epoch (returns at once).  The cross-process ordering needs a multi-GPU node.
hgks_status hgks_p2p_selftest(void) {
  return guard([&] {
    constexpr int n = 1000;
    double *src = nullptr, *dst = nullptr;
    int *list = nullptr;
    int2* map = nullptr;
    P2PFlags* fl = nullptr;
    auto cleanup = [&] {
      cudaFree(src); cudaFree(dst); cudaFree(list); cudaFree(map); cudaFree(fl);
    };
    try {
      CUDA_TRY(cudaMalloc(&src, sizeof(double) * QS * n));
      CUDA_TRY(cudaMalloc(&dst, sizeof(double) * QS * (n + 7)));
      CUDA_TRY(cudaMalloc(&list, sizeof(int) * n));
      CUDA_TRY(cudaMalloc(&map, sizeof(int2) * n));
      CUDA_TRY(cudaMalloc(&fl, sizeof(P2PFlags)));
      std::vector<double> hs((size_t)QS * n), hd((size_t)QS * (n + 7), -1.0);
      std::vector<int> hl(n);
      std::vector<int2> hm(n);
      for (size_t k = 0; k < hs.size(); ++k) hs[k] = 0.5 * (double)k + 1e-3;
      for (int j = 0; j < n; ++j) {
        hl[j] = (j * 37) % n;          // send rows in a scrambled order
        hm[j] = int2{3, 7 + (n - 1 - j)};  // receiver "rank 3", reversed rows after 7 others
      }
      CUDA_TRY(cudaMemcpy(src, hs.data(), hs.size() * sizeof(double), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(dst, hd.data(), hd.size() * sizeof(double), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(list, hl.data(), hl.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(map, hm.data(), hm.size() * sizeof(int2), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemset(fl, 0, sizeof(P2PFlags)));
      p64::PeerQ peer{};
      peer.q[3] = dst;
      p64::Launch::put(blocks(3 * n, 256), 0, src, list, map, n, peer);
      P2PSignal sg{};
      sg.dst[0] = &fl->arrived[5];
      sg.dst[1] = &fl->consumed[2];
      sg.n = 2;
      k_p2p_signal<<<1, 32>>>(sg, 7ull);
      CUDA_TRY(cudaGetLastError());
      P2PFlags h{};
      CUDA_TRY(cudaMemcpy(&h, fl, sizeof(P2PFlags), cudaMemcpyDeviceToHost));
      if (h.arrived[5] != 7 || h.consumed[2] != 7 || h.arrived[0] != 0)
        throw Error(HGKS_E_CUDA, "k_p2p_signal wrote wrong flags");
      // the fused put + release: rows again, flags to epoch 9, block counter back to 0
      P2PSignal sg2{};
      sg2.dst[0] = &fl->arrived[6];
      sg2.n = 1;
      p64::Launch::put_release(blocks(3 * n, 256), 0, src, list, map, n, peer, sg2, 9ull, &fl->put_blocks);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpy(&h, fl, sizeof(P2PFlags), cudaMemcpyDeviceToHost));
      if (h.arrived[6] != 9 || h.put_blocks != 0) throw Error(HGKS_E_CUDA, "k_put_release wrote wrong flags");
      P2PWait w{};
      w.src[0] = &fl->arrived[5];
      w.src[1] = &fl->consumed[2];
      w.n = 2;
      k_p2p_wait<<<1, 32>>>(w, 7ull);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaDeviceSynchronize());
      CUDA_TRY(cudaMemcpy(hd.data(), dst, hd.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int r = 0; r < 7; ++r)
        for (int v = 0; v < QS; ++v)
          if (hd[(size_t)r * QS + v] != -1.0) throw Error(HGKS_E_CUDA, "k_put wrote outside its rows");
      for (int j = 0; j < n; ++j)
        for (int v = 0; v < QS; ++v)
          if (hd[(size_t)(7 + n - 1 - j) * QS + v] != hs[(size_t)hl[j] * QS + v])
            throw Error(HGKS_E_CUDA, "k_put row " + std::to_string(j) + " differs");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

hgks_status hgks_nccl_selftest(void) {
  return guard([&] {
    Nccl& N = nccl();
    if (!N.h || !N.CommInitRank || !N.Send || !N.Recv || !N.AllReduce || !N.GroupStart || !N.GroupEnd)
      throw Error(HGKS_E_NCCL, "libnccl.so.2 not found or incomplete");
    ncclUniqueId id;
    NCCL_TRY(N.GetUniqueId(&id));
    ncclComm_t comm = nullptr;
    NCCL_TRY(N.CommInitRank(&comm, 1, id, 0));
    cudaStream_t st = nullptr, cs = nullptr;
    cudaEvent_t ev = nullptr;
    void* buf = nullptr;
    auto cleanup = [&] {
      if (st) cudaStreamSynchronize(st);
      if (cs) cudaStreamSynchronize(cs);
      if (buf) cudaFree(buf);
      if (ev) cudaEventDestroy(ev);
      if (st) cudaStreamDestroy(st);
      if (cs) cudaStreamDestroy(cs);
      if (comm && N.CommDestroy) N.CommDestroy(comm);
    };
    try {
      constexpr int n = 1000;
      CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_TRY(cudaMalloc(&buf, 2 * n * sizeof(double) + 2 * n * sizeof(float) + 64));
      double* d_src = (double*)buf;
      double* d_dst = d_src + n;
      float* f_src = (float*)(d_dst + n);
      float* f_dst = f_src + n;
      unsigned long long* bits = (unsigned long long*)(f_dst + n);
      std::vector<double> hs(n);
      std::vector<float> fs(n);
      for (int k = 0; k < n; ++k) hs[k] = fs[k] = 0.5f * k - 7.0f;
      const unsigned long long b0 = 0x3ff8000000000000ull;  // 1.5
      CUDA_TRY(cudaMemcpy(d_src, hs.data(), n * sizeof(double), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(f_src, fs.data(), n * sizeof(float), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(bits, &b0, sizeof(b0), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemset(d_dst, 0, n * sizeof(double)));
      CUDA_TRY(cudaMemset(f_dst, 0, n * sizeof(float)));
      // the halo pattern of exchange(): grouped send/recv on a comm stream, event back
      NCCL_TRY(N.GroupStart());
      NCCL_TRY(N.Send(d_src, n, ncclFloat64, 0, comm, cs));
      NCCL_TRY(N.Recv(d_dst, n, ncclFloat64, 0, comm, cs));
      NCCL_TRY(N.Send(f_src, n, ncclFloat32, 0, comm, cs));
      NCCL_TRY(N.Recv(f_dst, n, ncclFloat32, 0, comm, cs));
      NCCL_TRY(N.GroupEnd());
      CUDA_TRY(cudaEventRecord(ev, cs));
      CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
      // the dt pattern of allreduce_dt(): in-place min of the ordered bits
      NCCL_TRY(N.AllReduce(bits, bits, 1, ncclUint64, ncclMin, comm, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      std::vector<double> hd(n);
      std::vector<float> fd(n);
      unsigned long long b1 = 0;
      CUDA_TRY(cudaMemcpy(hd.data(), d_dst, n * sizeof(double), cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(fd.data(), f_dst, n * sizeof(float), cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(&b1, bits, sizeof(b1), cudaMemcpyDeviceToHost));
      if (hd != hs || fd != fs) throw Error(HGKS_E_NCCL, "NCCL self send/recv returned wrong data");
      if (b1 != b0) throw Error(HGKS_E_NCCL, "NCCL allreduce(min, uint64) returned wrong data");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

hgks_status hgks_group_step(hgks_solver* const* ss, int32_t n, int32_t n_steps, double t_stop) {
  return guard([&] {
    if (!ss || n < 1 || n > kMaxGroup) throw Error(HGKS_E_ARG, "bad group size");
    for (int k = 0; k < n; ++k) {
      if (!ss[k] || ss[k]->transport != HGKS_TRANSPORT_LOOPBACK || ss[k]->n_ranks != n || ss[k]->rank != k)
        throw Error(HGKS_E_ARG, "hgks_group_step needs the loopback solvers of ranks 0..n-1 in order");
      if (ss[k]->stream != ss[0]->stream || ss[k]->device != ss[0]->device || ss[k]->fp32 != ss[0]->fp32)
        throw Error(HGKS_E_ARG, "loopback solvers must share one device and stream");
    }
    hgks_solver* s0 = ss[0];
    GroupCtrl gc;
    gc.n = n;
    for (int k = 0; k < n; ++k) gc.c[k] = ss[k]->d.ctrl;
    auto group_min = [&] { launch(s0, "k_group_min", [&] { k_group_min<<<1, 32, 0, s0->stream>>>(gc); }); };
    // ghost rows: fused put of every rank's send rows into its receivers (f3)
    build_put_map(ss, n);
    group_min();
    for (int step = 0; step < n_steps; ++step) {
      for (int k = 0; k < n; ++k)
        launch(ss[k], "k_step_begin", [&] {
          k_step_begin<<<1, 1, 0, s0->stream>>>(ss[k]->d.ctrl, ss[k]->cfg.cfl, ss[k]->cfg.fixed_dt, t_stop);
        });
      for (int st = 1; st <= 2; ++st) {
        for (int k = 0; k < n; ++k) HGKS_DISPATCH(ss[k], put, ss, k, n);
        for (int k = 0; k < n; ++k) HGKS_DISPATCH(ss[k], stage_early, ss[k], st);
        for (int k = 0; k < n; ++k) HGKS_DISPATCH(ss[k], stage_late, ss[k], st);
      }
      group_min();
    }
  });
}

hgks_status hgks_mesh_plan(const hgks_mesh* mc, int32_t rank, int64_t* l2g, int32_t* peers, int64_t* send_off,
                           int64_t* send_cnt, int32_t* send_list, int64_t* recv_off, int64_t* recv_cnt) {
  return guard([&] {
    if (!mc) throw Error(HGKS_E_ARG, "null mesh");
    hgks_mesh* m = const_cast<hgks_mesh*>(mc);
    const RankPlan& rp = m->plan(rank);
    if (l2g) std::copy(rp.l2g.begin(), rp.l2g.end(), l2g);
    if (peers) std::copy(rp.peers.begin(), rp.peers.end(), peers);
    if (send_off) std::copy(rp.send_off.begin(), rp.send_off.end(), send_off);
    if (send_cnt) std::copy(rp.send_cnt.begin(), rp.send_cnt.end(), send_cnt);
    if (send_list) std::copy(rp.send_list.begin(), rp.send_list.end(), send_list);
    if (recv_off) std::copy(rp.recv_off.begin(), rp.recv_off.end(), recv_off);
    if (recv_cnt) std::copy(rp.recv_cnt.begin(), rp.recv_cnt.end(), recv_cnt);
  });
}

// ---- f3: cross-process fused halo put (HGKS_TRANSPORT_P2P) ----
namespace {
struct P2PBlob {  // HGKS_P2P_HANDLE_BYTES
  cudaIpcMemHandle_t mem;  // the allocation holding this rank's workspace
  uint64_t off_Q, off_flags;  // byte offsets of Q and the flags from the allocation base
  int32_t rank, device;
  char bus_id[16];         // PCI bus id of the device (unique across processes, unlike the ordinal)
  RecvTab recv;            // where this rank keeps each peer's ghost rows (the senders' put map)
  uint8_t pad[HGKS_P2P_HANDLE_BYTES - sizeof(cudaIpcMemHandle_t) - 16 - 8 - 16 - sizeof(RecvTab)];
};
static_assert(sizeof(P2PBlob) == HGKS_P2P_HANDLE_BYTES, "blob size");

// base of the device allocation containing p (driver API, resolved at run time)
char* alloc_base(void* p) {
  typedef int (*Fn)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    return h ? (Fn)dlsym(h, "cuMemGetAddressRange_v2") : (Fn) nullptr;
  }();
  if (!fn) throw Error(HGKS_E_CUDA, "cuMemGetAddressRange_v2 not found in libcuda.so.1");
  unsigned long long base = 0;
  size_t size = 0;
  if (fn(&base, &size, (unsigned long long)(uintptr_t)p) != 0) throw Error(HGKS_E_CUDA, "cuMemGetAddressRange failed");
  return reinterpret_cast<char*>(base);
}
}  // namespace

hgks_status hgks_p2p_export(const hgks_solver* s, uint8_t* out) {
  return guard([&] {
    if (!s || !out) throw Error(HGKS_E_ARG, "null argument");
    if (s->transport != HGKS_TRANSPORT_P2P) throw Error(HGKS_E_ARG, "solver transport is not HGKS_TRANSPORT_P2P");
    CUDA_TRY(cudaSetDevice(s->device));
    P2PBlob b{};
    char* base = alloc_base(s->d.Q);
    CUDA_TRY(cudaIpcGetMemHandle(&b.mem, base));
    b.off_Q = (uint64_t)((char*)s->d.Q - base);
    b.off_flags = (uint64_t)((char*)s->d.flags - base);
    b.rank = s->rank;
    b.device = s->device;
    CUDA_TRY(cudaDeviceGetPCIBusId(b.bus_id, (int)sizeof(b.bus_id), s->device));
    b.recv = recv_tab(*s->rp);
    std::memcpy(out, &b, sizeof(b));
  });
}

hgks_status hgks_p2p_connect(hgks_solver* s, const uint8_t* blobs) {
  return guard([&] {
    if (!s || !blobs) throw Error(HGKS_E_ARG, "null argument");
    if (s->transport != HGKS_TRANSPORT_P2P) throw Error(HGKS_E_ARG, "solver transport is not HGKS_TRANSPORT_P2P");
    if (s->p2p_ready) throw Error(HGKS_E_STATE, "already connected");
    CUDA_TRY(cudaSetDevice(s->device));
    const RankPlan& rp = *s->rp;
    // the receivers' ghost ranges come with their blobs: no peer plan is built here
    std::vector<P2PBlob> all_blobs(s->n_ranks);
    for (int p = 0; p < s->n_ranks; ++p) std::memcpy(&all_blobs[p], blobs + (size_t)p * HGKS_P2P_HANDLE_BYTES, sizeof(P2PBlob));
    std::vector<int2> dst = put_map(rp, s->rank, [&](int p) -> const RecvTab& { return all_blobs[p].recv; });
    char my_bus[16];
    CUDA_TRY(cudaDeviceGetPCIBusId(my_bus, (int)sizeof(my_bus), s->device));
    std::vector<int> to;
    for (const int2& d : dst) to.push_back(d.x);
    std::sort(to.begin(), to.end());
    to.erase(std::unique(to.begin(), to.end()), to.end());
    std::vector<int> from;
    for (size_t ip = 0; ip < rp.peers.size(); ++ip)
      if (rp.recv_cnt[ip] > 0) from.push_back(rp.peers[ip]);
    std::vector<int> all = to;
    all.insert(all.end(), from.begin(), from.end());
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    for (int p : all) {
      P2PBlob b;
      std::memcpy(&b, blobs + (size_t)p * HGKS_P2P_HANDLE_BYTES, sizeof(b));
      if (b.rank != p) throw Error(HGKS_E_ARG, "blob " + std::to_string(p) + " belongs to rank " + std::to_string(b.rank));
      if (std::strncmp(b.bus_id, my_bus, sizeof(my_bus)) == 0)
        throw Error(HGKS_E_ARG, "HGKS_TRANSPORT_P2P needs one GPU per rank (rank " + std::to_string(p) +
                                    " is on this rank's device " + std::string(my_bus) + ")");
      int peer_dev = -1, can = 0;
      if (cudaDeviceGetByPCIBusId(&peer_dev, b.bus_id) == cudaSuccess) {
        CUDA_TRY(cudaDeviceCanAccessPeer(&can, s->device, peer_dev));
        if (!can) throw Error(HGKS_E_ARG, "no peer access from " + std::string(my_bus) + " to " + b.bus_id);
      }
      void* base = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&base, b.mem, cudaIpcMemLazyEnablePeerAccess));
      s->peer_base[p] = base;
      s->peer_Q[p] = (char*)base + b.off_Q;
      s->peer_flags[p] = reinterpret_cast<P2PFlags*>((char*)base + b.off_flags);
    }
    if (!dst.empty())
      CUDA_TRY(cudaMemcpy(s->d.put_dst, dst.data(), dst.size() * sizeof(int2), cudaMemcpyHostToDevice));
    s->put_to = to;
    s->recv_from = from;
    s->p2p_ready = true;
  });
}

hgks_status hgks_mesh_put_map(const hgks_mesh* mc, int32_t rank, int32_t* recv_rank, int32_t* recv_row) {
  return guard([&] {
    if (!mc || !recv_rank || !recv_row) throw Error(HGKS_E_ARG, "null argument");
    hgks_mesh* m = const_cast<hgks_mesh*>(mc);
    const std::vector<int2> dst = put_map_mesh(m, rank);
    for (size_t j = 0; j < dst.size(); ++j) {
      recv_rank[j] = dst[j].x;
      recv_row[j] = dst[j].y;
    }
  });
}

hgks_status hgks_launch_count(const hgks_solver* s, int64_t* launches) {
  if (!s || !launches) return HGKS_E_ARG;
  *launches = s->launches;
  return HGKS_OK;
}

}  // extern "C"
