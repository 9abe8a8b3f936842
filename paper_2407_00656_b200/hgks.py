"""Thin Python binding of libhgks.so (include/hgks.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of csrc/.  PyTorch provides
device memory (the workspace tensor), the stream and torch.distributed (used
only to broadcast the NCCL unique id).  There is no CPU fallback: if the
library or a CUDA device is missing, these calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)

HGKS_TET, HGKS_PRISM, HGKS_HEX = 4, 6, 8
ERRORS = {0: "OK", 1: "E_ARG", 2: "E_MESH", 3: "E_STENCIL", 4: "E_CUDA", 5: "E_NCCL", 6: "E_POSITIVITY",
          7: "E_STATE"}

# every symbol include/hgks.h declares (checked by tests/test_abi.py)
EXPORTS = ["hgks_mesh_create", "hgks_mesh_destroy", "hgks_mesh_info", "hgks_workspace_size", "hgks_init",
           "hgks_destroy", "hgks_step", "hgks_set_state", "hgks_get_state", "hgks_get_state_async",
           "hgks_sync", "hgks_debug_residual",
           "hgks_set_profiling", "hgks_kernel_times", "hgks_launch_count", "hgks_nccl_unique_id", "hgks_nccl_selftest", "hgks_group_step", "hgks_mesh_plan", "hgks_mesh_put_map", "hgks_p2p_export", "hgks_p2p_connect", "hgks_p2p_selftest",
           "hgks_last_error", "hgks_version"]
TRANSPORT_NCCL, TRANSPORT_LOOPBACK, TRANSPORT_P2P = 0, 1, 2
P2P_HANDLE_BYTES = 448


class MeshDesc(C.Structure):
    _fields_ = [("xyz", _dp), ("n_nodes", C.c_int64), ("cell_type", _i8p), ("cell_nodes", _i64p),
                ("n_cells", C.c_int64), ("periodic_origin", C.c_double * 3), ("periodic_length", C.c_double * 3),
                ("bface_nodes", _i64p), ("bface_tag", _i32p), ("n_bfaces", C.c_int64), ("n_ranks", C.c_int32),
                ("cell_part", _i32p), ("rank_only", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("gamma", C.c_double), ("cfl", C.c_double), ("fixed_dt", C.c_double), ("tau_mode", C.c_int32),
                ("c1", C.c_double), ("mu_inf", C.c_double), ("t_inf", C.c_double), ("mu_exp", C.c_double),
                ("eps", C.c_double), ("omega_pow", C.c_int32), ("freestream", C.c_double * 5),
                ("precision", C.c_int32), ("dq0_mode", C.c_int32), ("prandtl", C.c_double)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("n_ranks", C.c_int32), ("device", C.c_int32), ("transport", C.c_int32),
                ("nccl_id", C.c_uint8 * 128)]


class MeshStats(C.Structure):
    _fields_ = [("n_cells_global", C.c_int64), ("n_owned", C.c_int64), ("n_ghost", C.c_int64),
                ("ghost_layer", C.c_int64 * 3), ("n_bghost", C.c_int64), ("n_faces", C.c_int64),
                ("n_faces_bc", C.c_int64), ("stencil_min", C.c_int32), ("stencil_max", C.c_int32),
                ("n_sub", C.c_int32), ("n_peers", C.c_int32), ("send_cells", C.c_int64), ("recv_cells", C.c_int64),
                ("edge_cut", C.c_int64), ("n_early_cells", C.c_int64), ("n_early_faces", C.c_int64),
                ("edge_cut_rcb", C.c_int64), ("rank_cut_faces", C.c_int64)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if name == "ghost_layer" else int(v)
        return d


class StepInfo(C.Structure):
    _fields_ = [("steps_done", C.c_int64), ("t", C.c_double), ("last_dt", C.c_double), ("fallbacks", C.c_int64)]


class HgksError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib(build_if_needed: bool = True):
    """Load libhgks.so (building it in-tree with nvcc when sources changed)."""
    global _lib
    if _lib is None:
        if build_if_needed and _build.needs_build():
            _build.build()
        path = os.environ.get("HGKS_LIB", _build.LIB)  # experiments may point at another build
        if not os.path.exists(path):
            raise RuntimeError(f"libhgks.so missing at {path}: run __graft_entry__.build()")
        L = C.CDLL(path)
        L.hgks_last_error.restype = C.c_char_p
        L.hgks_version.restype = C.c_char_p
        L.hgks_mesh_create.argtypes = [C.POINTER(MeshDesc), C.POINTER(C.c_void_p)]
        L.hgks_mesh_destroy.argtypes = [C.c_void_p]
        L.hgks_mesh_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(MeshStats)]
        L.hgks_workspace_size.argtypes = [C.c_void_p, C.POINTER(Config), C.c_int32, C.POINTER(C.c_size_t)]
        L.hgks_init.argtypes = [C.c_void_p, C.POINTER(Config), C.POINTER(Dist), C.c_void_p, C.c_size_t, C.c_void_p,
                                _dp, C.POINTER(C.c_void_p)]
        L.hgks_destroy.argtypes = [C.c_void_p]
        L.hgks_step.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.POINTER(StepInfo)]
        L.hgks_set_state.argtypes = [C.c_void_p, C.c_void_p, C.c_double]
        L.hgks_get_state.argtypes = [C.c_void_p, C.c_void_p, _i64p, _dp]
        L.hgks_debug_residual.argtypes = [C.c_void_p, _dp, C.c_double, _dp, _dp]
        L.hgks_set_profiling.argtypes = [C.c_void_p, C.c_int32]
        L.hgks_kernel_times.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, _i64p, _dp, _i32p]
        L.hgks_launch_count.argtypes = [C.c_void_p, _i64p]
        L.hgks_nccl_unique_id.argtypes = [C.c_void_p]
        L.hgks_p2p_export.argtypes = [C.c_void_p, C.c_void_p]
        L.hgks_p2p_connect.argtypes = [C.c_void_p, C.c_void_p]
        L.hgks_group_step.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_double]
        L.hgks_mesh_plan.argtypes = [C.c_void_p, C.c_int32, _i64p, _i32p, _i64p, _i64p, _i32p, _i64p, _i64p]
        L.hgks_mesh_put_map.argtypes = [C.c_void_p, C.c_int32, _i32p, _i32p]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise HgksError(rc, lib().hgks_last_error().decode())


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


@dataclass
class SolverConfig:
    gamma: float = 1.4
    cfl: float = 0.3
    fixed_dt: float = 0.0
    tau_mode: int = 0
    c1: float = 1.0
    mu_inf: float = 0.0
    t_inf: float = 1.0
    mu_exp: float = 0.7
    eps: float | None = None  # WENO epsilon; None: 1e-10 (fp64) / 1e-6 (fp32), reading R27
    omega_pow: int = 1
    freestream: tuple = (1.0, 0.0, 0.0, 0.0, 1.0 / 1.4)
    precision: int = 64  # 64: fp64 parity path; 32: FP32 variant
    dq0_mode: int = 0    # equilibrium slopes: 0 average (R9), 1 kinetic (R9k), 2 gamma-weighted (R9s)
    prandtl: float = 1.0  # Pr of the heat-flux correction (R29); 1 = none (BGK)

    def eps_value(self) -> float:
        if self.eps is not None:
            return self.eps
        return 1e-10 if self.precision == 64 else 1e-6

    def c(self) -> Config:
        return Config(self.gamma, self.cfl, self.fixed_dt, self.tau_mode, self.c1, self.mu_inf, self.t_inf,
                      self.mu_exp, self.eps_value(), self.omega_pow, (C.c_double * 5)(*self.freestream), self.precision,
                      self.dq0_mode, self.prandtl)


def p2p_selftest() -> None:
    """k_put / k_p2p_signal / k_p2p_wait mechanics on one device (hgks_p2p_selftest)."""
    _check(lib().hgks_p2p_selftest())


def nccl_selftest() -> None:
    """One-rank NCCL communicator doing the calls of a multi-rank step (diagnostic)."""
    _check(lib().hgks_nccl_selftest())


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().hgks_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Mesh:
    """hgks_mesh: host setup (geometry, faces, stencils, LSQ operators, partition)."""

    def __init__(self, mi, n_ranks: int = 1, cell_part=None, rank: int | None = None):
        """rank: build only that rank's region (one process per GPU; O(owned + ghosts) host
        memory); None: the whole mesh and every rank's plan."""
        L = lib()
        self._keep = [np.ascontiguousarray(mi.xyz, np.float64), np.ascontiguousarray(mi.cell_type, np.int8),
                      np.ascontiguousarray(mi.cell_nodes, np.int64),
                      np.ascontiguousarray(mi.bface_nodes, np.int64).reshape(-1, 4),
                      np.ascontiguousarray(mi.bface_tag, np.int32)]
        xyz, ct, cn, bf, bt = self._keep
        part = None
        if cell_part is not None:
            part = np.ascontiguousarray(cell_part, np.int32)
            self._keep.append(part)
        d = MeshDesc(_p(xyz), xyz.shape[0], _p(ct, _i8p), _p(cn, _i64p), cn.shape[0],
                     (C.c_double * 3)(*mi.periodic_origin), (C.c_double * 3)(*mi.periodic_length),
                     _p(bf, _i64p), _p(bt, _i32p), bf.shape[0], n_ranks,
                     _p(part, _i32p) if part is not None else None, 0 if rank is None else rank + 1)
        h = C.c_void_p()
        _check(L.hgks_mesh_create(C.byref(d), C.byref(h)))
        self.h = h
        self.n_ranks = n_ranks
        self.n_cells = int(cn.shape[0])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hgks_mesh_destroy(self.h)
            self.h = None

    def info(self, rank: int = 0) -> dict:
        st = MeshStats()
        _check(lib().hgks_mesh_info(self.h, rank, C.byref(st)))
        return st.as_dict()

    def plan(self, rank: int = 0) -> dict:
        """Partition plan of one rank (hgks_mesh_plan): local->global ids and per-peer exchange lists."""
        st = self.info(rank)
        nl = st["n_owned"] + st["n_ghost"]
        npr = st["n_peers"]
        l2g = np.zeros(nl, np.int64)
        peers = np.zeros(max(npr, 1), np.int32)
        so = np.zeros(max(npr, 1), np.int64); sc = np.zeros(max(npr, 1), np.int64)
        ro = np.zeros(max(npr, 1), np.int64); rc = np.zeros(max(npr, 1), np.int64)
        sl = np.zeros(max(st["send_cells"], 1), np.int32)
        _check(lib().hgks_mesh_plan(self.h, rank, _p(l2g, _i64p), _p(peers, _i32p), _p(so, _i64p), _p(sc, _i64p),
                                    _p(sl, _i32p), _p(ro, _i64p), _p(rc, _i64p)))
        return dict(n_owned=st["n_owned"], l2g=l2g, peers=peers[:npr], send_off=so[:npr], send_cnt=sc[:npr],
                    send_list=sl[:st["send_cells"]], recv_off=ro[:npr], recv_cnt=rc[:npr])

    def put_map(self, rank: int = 0):
        """Fused-put destinations of rank's send rows (hgks_mesh_put_map): (receiver rank, receiver row)."""
        n = self.info(rank)["send_cells"]
        rr = np.zeros(max(n, 1), np.int32)
        row = np.zeros(max(n, 1), np.int32)
        _check(lib().hgks_mesh_put_map(self.h, rank, _p(rr, _i32p), _p(row, _i32p)))
        return rr[:n], row[:n]

    def workspace_size(self, cfg: SolverConfig, rank: int = 0) -> int:
        n = C.c_size_t()
        _check(lib().hgks_workspace_size(self.h, C.byref(cfg.c()), rank, C.byref(n)))
        return int(n.value)


def group_step(solvers, n_steps: int, t_stop: float = 0.0):
    """Advance loopback solvers of ranks 0..n-1 together (hgks_group_step)."""
    arr = (C.c_void_p * len(solvers))(*[s.h for s in solvers])
    _check(lib().hgks_group_step(arr, len(solvers), n_steps, t_stop))


class Solver:
    """hgks_solver on one CUDA device.  ``Q0``: [n_cells_global, 5] float64 (caller order)."""

    def __init__(self, mesh: Mesh, Q0, cfg: SolverConfig | None = None, device=None, rank: int = 0,
                 nccl_id: bytes | None = None, transport: int = TRANSPORT_NCCL):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("hgks needs a CUDA device (no CPU fallback)")
        self.cfg = cfg or SolverConfig()
        self.mesh = mesh
        self._inflight = []  # host buffers of enqueued copies (kept alive until sync)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        torch.cuda.set_device(self.device)
        nbytes = mesh.workspace_size(self.cfg, rank)
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        ptr = (base + 255) // 256 * 256
        self.stream = torch.cuda.current_stream(self.device)
        Q0 = np.ascontiguousarray(Q0, np.float64)
        dist = None
        if mesh.n_ranks > 1:
            nid = nccl_id if nccl_id is not None else bytes(128)
            dist = Dist(rank, mesh.n_ranks, self.device.index, transport, (C.c_uint8 * 128)(*nid))
        h = C.c_void_p()
        _check(lib().hgks_init(mesh.h, C.byref(self.cfg.c()), C.byref(dist) if dist else None, C.c_void_p(ptr),
                               nbytes, C.c_void_p(self.stream.cuda_stream), _p(Q0), C.byref(h)))
        self.h = h
        self.rank = rank
        self.n_owned = mesh.info(rank)["n_owned"]

    def p2p_export(self) -> bytes:
        """This rank's HGKS_TRANSPORT_P2P blob (hgks_p2p_export)."""
        buf = (C.c_uint8 * P2P_HANDLE_BYTES)()
        _check(lib().hgks_p2p_export(self.h, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def p2p_connect(self, blobs):
        """Map the peers' workspaces (hgks_p2p_connect); ``blobs``: every rank's blob in rank order."""
        raw = b"".join(blobs)
        assert len(raw) == P2P_HANDLE_BYTES * self.mesh.n_ranks
        buf = (C.c_uint8 * len(raw)).from_buffer_copy(raw)
        _check(lib().hgks_p2p_connect(self.h, C.cast(buf, C.c_void_p)))

    def p2p_connect_dist(self):
        """All-gather the blobs over torch.distributed and connect (collective)."""
        import torch.distributed as dist
        blobs = [None] * self.mesh.n_ranks
        dist.all_gather_object(blobs, self.p2p_export())
        self.p2p_connect(blobs)

    def close(self):
        if getattr(self, "h", None):
            _check(lib().hgks_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, n_steps: int = 1, t_stop: float = 0.0, info: bool = True):
        si = StepInfo()
        _check(lib().hgks_step(self.h, n_steps, t_stop, C.byref(si) if info else None))
        if info:
            return dict(steps_done=int(si.steps_done), t=float(si.t), last_dt=float(si.last_dt),
                        fallbacks=int(si.fallbacks))
        return None

    def set_state(self, Q, t: float = 0.0):
        """Q: numpy [n,5] float64 or a (pinned) CPU torch tensor.  Asynchronous: the
        buffer is kept alive here until the next sync()/get_state()."""
        if not hasattr(Q, "data_ptr"):
            Q = np.ascontiguousarray(Q, np.float64)
        self._inflight.append(Q)
        ptr = Q.data_ptr() if hasattr(Q, "data_ptr") else Q.ctypes.data
        _check(lib().hgks_set_state(self.h, C.c_void_p(ptr), t))

    def get_state_async(self, out):
        """Enqueue the download of the current state into ``out`` (pinned CPU tensor or
        numpy [n_owned,5] float64, ascending global id); valid after sync()."""
        self._inflight.append(out)
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        _check(lib().hgks_get_state_async(self.h, C.c_void_p(ptr)))

    def sync(self):
        _check(lib().hgks_sync(self.h))
        self._inflight.clear()

    def get_state(self, out=None):
        """Owned cells in ascending global id -> (Q [n_owned,5], gid, t).  ``out`` may be a pinned tensor."""
        t = C.c_double()
        gid = np.zeros(self.n_owned, np.int64)
        if out is None:
            Q = np.zeros((self.n_owned, 5))
            _check(lib().hgks_get_state(self.h, C.c_void_p(Q.ctypes.data), _p(gid, _i64p), C.byref(t)))
            self._inflight.clear()
            return Q, gid, t.value
        _check(lib().hgks_get_state(self.h, C.c_void_p(out.data_ptr()), None, C.byref(t)))
        self._inflight.clear()
        return out, None, t.value

    def residual(self, Q, dt: float):
        Q = np.ascontiguousarray(Q, np.float64)
        L = np.zeros_like(Q)
        dL = np.zeros_like(Q)
        _check(lib().hgks_debug_residual(self.h, _p(Q), dt, _p(L), _p(dL)))
        return L, dL

    def set_profiling(self, on: bool):
        _check(lib().hgks_set_profiling(self.h, 1 if on else 0))

    def kernel_times(self) -> dict:
        cap = 64
        names = (C.c_char * 32 * cap)()
        launches = np.zeros(cap, np.int64)
        ms = np.zeros(cap)
        n = C.c_int32()
        _check(lib().hgks_kernel_times(self.h, cap, C.cast(names, C.c_void_p), _p(launches, _i64p), _p(ms),
                                       C.byref(n)))
        out = {}
        for k in range(n.value):
            nm = bytes(names[k]).split(b"\0", 1)[0].decode()
            out[nm] = dict(launches=int(launches[k]), ms=float(ms[k]))
        return out

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().hgks_launch_count(self.h, C.byref(n)))
        return int(n.value)
