"""Benchmark: fp64 cell-updates/s of the HGKS hot path on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c5|c2|c3|c4]

One step = one full S2O4 step (2 stages of halo exchange + WENO reconstruction
+ face flux + update, plus the CFL min) over every cell.  Default workload: the
largest single-GPU configuration of BASELINE.json, configs[4] -- the 110^3 Kuhn
box, 7,986,000 periodic tets per GPU, tau = 0, CFL 0.3, accuracy-test IC.  N > 1
(torchrun, one process per GPU): weak scaling, one 110^3 block per GPU (box
extended along x/y/z, RCB partition, NCCL halo exchange + allreduce-min).
--workload c2 (48^3, configs[1]), c3/c4 (sphere shells, configs[2]/[3]) are
the other configurations.

--impl reference times the CPU oracle (oracle/) on the box's host cores on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BLOCK = 48            # cubes per axis per GPU block (configs[1] top size)
N_BLOCK_C5 = 110        # configs[4]: ~8M tets per GPU (110^3 cubes x 6)
GAMMA = 1.4
CFL = 0.3
METRIC = "fp64 cell-updates/sec at 1/2/4/8 B200; % HBM/FP64 roofline"
UNIT = "cell-updates/s"


def box_dims(n_gpus: int, nb: int = N_BLOCK):
    """Weak-scaling box: n_gpus blocks of nb^3 cubes (factor 2 per axis, x first)."""
    dims = [1, 1, 1]
    k, ax = n_gpus, 0
    while k > 1:
        if k % 2:
            dims[ax] *= k
            break
        dims[ax] *= 2
        k //= 2
        ax = (ax + 1) % 3
    return [d * nb for d in dims]


def peaks(precision=64):
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = None
    if os.path.exists(path):
        hbm = json.load(open(path)).get("hbm_gbs")
    src = "MEASURED_PEAKS.json" if hbm else "fallback B200_PROFILING.md"
    pk = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    key = "fp64_tflops" if precision == 64 else "fp32_tflops"
    kind = "DFMA" if precision == 64 else "FFMA"
    return (hbm or 6650.0), src, pk[key], (f"builder-measured: profiles/fp64_peak.json {key} ({kind}-chain "
                                           f"microbenchmark on this pool; not in MEASURED_PEAKS.json)")


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML polled every 5 ms from a thread (so even a few-hundred-millisecond timed region
    carries its own record; the GPU is found by its PCI bus id, robust to
    CUDA_VISIBLE_DEVICES); nvidia-smi -lms 100 if NVML is unavailable."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, sm_max_mhz, {reason names})
        self.proc = None
        self.stop = threading.Event()
        self.src = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(self.index)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)

    def _poll_nvml(self, nv, h):
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))
            time.sleep(0.005)

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]),
                                  {self.REASONS[k] for k in range(4) if parts[2 + k].lower() == "active"}))

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.src = "nvml 5 ms"
        except Exception:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read_smi, daemon=True)
                self.src = "nvidia-smi 100 ms"
            except Exception:
                return self
        self.t.start()
        t0 = time.time()
        while not self.rows and time.time() - t0 < 10:  # sampler is live before the timed region
            time.sleep(0.01)
        self.rows.clear()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.src:
            self.t.join(timeout=2)

    def summary(self):
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0, "source": self.src}
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(set().union(*[r[2] for r in rows])), "samples": len(rows), "source": self.src}


# algorithmic bytes / flops per unit, tets
RECON_NE = False  # csrc/internal.h HGKS_RECON_NE (default build 0: streamed pseudo-inverse)


def recon_bytes_per_cell(K=14, M=4, NM=6, rs=8, ne=RECON_NE):
    """Algorithmic bytes per reconstructed cell.  rs: bytes of the working
    precision (8 fp64, 4 for the FP32 variant).  ne: P_0 by normal equations -- the 9x9 inverse
    Cholesky factor (45 entries + 1 pad) instead of the 9 x K pseudo-inverse, one image code per
    member, and the cell's own row of member geometry (centroid, M2: 10 values; each row is
    read at least once per launch, its other uses hit L2)."""
    op = ((46 if ne else 9 * K) + M * 3 * NM) * rs  # LSQ operators
    idx = K * 4 + M * NM * 1 + 4       # stencil ids, sub-stencil slots, recon cell id
    if NM == 7:
        idx += 1                       # hybrid layouts: the cell's sub-stencil count
    if ne:
        idx += K                       # periodic image codes of the members
    geo = 8 * rs                       # V^{2/3}, V^{4/3}, M2
    if ne:
        geo += 10 * rs                 # member geometry row (centroid, M2, pad)
    q = 5 * rs                         # the cell's own state (neighbours: each state read once overall)
    rec = 50 * rs                      # effective-polynomial record written
    return op + idx + geo + q + rec


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_problem(workload: str, N: int):
    """The oracle's copy of a bench workload at a bounded size: Kuhn box N^3 (c2/c5, the same
    per-cell work at any box size) or sphere shell 12 N^3 (c3/c4)."""
    from oracle import oracle as O
    from paper_2407_00656_b200 import workloads as W
    if workload in ("c2", "c5"):
        mi = W.kuhn_box(N)
        return mi, W.advection_ic(mi, gamma=GAMMA), O.OracleConfig(cfl=CFL), f"{N}^3 Kuhn box ({6 * N ** 3} tets)"
    ma, re, _ = SPHERE[workload]
    mi = sphere_mesh(workload, N)
    Q0 = W.uniform_state(mi.n_cells, 1.0, (ma, 0.0, 0.0), 1.0 / GAMMA, gamma=GAMMA)
    cfg = O.OracleConfig(cfl=sphere_cfl(workload), tau_mode=1, mu_inf=ma / re, c1=1.0, t_inf=1.0 / GAMMA,
                         freestream=(1.0, ma, 0.0, 0.0, 1.0 / GAMMA))
    what = (f"hybrid tet/prism sphere N = {N} ({mi.n_cells} cells, Ma {ma}, Re {re})" if workload == "c3h" else
            f"sphere shell 12x{N}^3 ({12 * N ** 3} hexes, Ma {ma}, Re {re})")
    return mi, Q0, cfg, what


def cpu_oracle_rate(workload: str, N: int, steps: int, threads: int):
    from oracle import oracle as O
    mi, Q0, cfg, what = oracle_problem(workload, N)
    m = O.OracleMesh(mi)
    s = O.OracleSolver(m, Q0, cfg, threads=threads)
    t0 = time.perf_counter()
    s.step(steps)
    dt = time.perf_counter() - t0
    return m.n_cells * steps / dt, dt, what


# bounded oracle samples per workload family: (all cores N, one core N); the oracle's cost per
# cell does not depend on the box size, so a smaller box of the same family is the same work
CPU_SAMPLE = {"c2": (48, 12), "c5": (48, 12), "c3": (12, 5), "c4": (12, 5), "c3h": (20, 6)}


def cpu_baseline(workload: str):
    threads = len(os.sched_getaffinity(0))
    n_all, n_one = CPU_SAMPLE[workload]
    rate, secs, what = cpu_oracle_rate(workload, n_all, 1, threads)
    rate1, secs1, what1 = cpu_oracle_rate(workload, n_one, 1, 1)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"1 oracle step of the {what}, same workload family and per-cell work, {secs:.1f} s on "
                      f"{threads} threads",
            "one_thread": {"value": rate1, "unit": UNIT, "cores": 1,
                           "sample": f"1 oracle step of the {what1}, {secs1:.1f} s on 1 thread"},
            "cpu_model": cpu_model()}


SPHERE = {"c3": (0.2535, 118.0, 35), "c4": (1.5, 300.0, 70), "c3h": (0.2535, 118.0, 20)}


def sphere_mesh(workload: str, n: int):
    """c3/c4: hex cubed-sphere shell 12 n^3; c3h: the hybrid tet/prism sphere of BASELINE.json
    configs[2] ("~0.5M mixed tet/prism cells"): prisms in the first n/2 of 2n radial layers,
    tets outside (n = 20: 480,000 cells)."""
    from paper_2407_00656_b200 import workloads as W
    return W.sphere_hybrid(n, prism_layers=n // 2) if workload == "c3h" else W.sphere_shell(n)


def sphere_cfl(workload: str) -> float:
    return 0.3 if workload == "c3h" else 0.5  # tets in the mesh: the tet CFL (R6)


def workload_config(workload: str, world: int, box: int = 0, jitter: float = 0.0):
    """(config dict, scaling, recon layout) of a bench workload; no mesh is built here."""
    if workload in ("c2", "c5"):
        nb = N_BLOCK if workload == "c2" else N_BLOCK_C5
        if box > 0 and workload == "c2":
            nb = box
        nx, ny, nz = box_dims(world, nb)
        wl = (f"configs[1]{' top size' if nb == N_BLOCK else ''}: {nb}^3 Kuhn box per GPU, 6 tets/cube, periodic, "
              f"tau=0, CFL {CFL}" if workload == "c2" else
              f"configs[4]: {nb}^3 Kuhn box ({6 * nb ** 3} tets) per GPU, periodic, tau=0, CFL {CFL}")
        cfg = {"workload": wl, "cells": 6 * nx * ny * nz, "box_cubes": [nx, ny, nz], "block_cubes": nb}
        if jitter > 0:
            cfg["workload"] += f", nodes jittered U[-{jitter}h, {jitter}h] (seed 656)"
            cfg["jitter"] = jitter
        return cfg, "weak", (14, 4, 6)
    ma, re, n = SPHERE[workload]
    if workload == "c3h":
        wl = (f"configs[2]: hybrid tet/prism sphere, cubed-sphere N = {n}, {n // 2} prism layers + "
              f"{2 * n - n // 2} tet layers ({6 * n * n * (2 * (n // 2) + 6 * (2 * n - n // 2))} cells), Ma {ma}, "
              f"Re {re}, NS collision time, wall + farfield, CFL 0.3, free-stream start")
        return ({"workload": wl, "cells": 6 * n * n * (2 * (n // 2) + 6 * (2 * n - n // 2)), "sphere_N": n},
                "strong", (24, 6, 7))
    wl = (f"configs[{2 if workload == 'c3' else 3}]: sphere shell 12x{n}^3 hexes, Ma {ma}, Re {re}, "
          f"NS collision time, wall + farfield, CFL 0.5, free-stream start")
    return {"workload": wl, "cells": 12 * n ** 3, "sphere_N": n}, "strong", (24, 8, 3)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    from oracle import oracle as O
    # bounded sample: every timed step is one full oracle step of the same workload family on a
    # smaller box, sized so the whole --steps/--warmup run stays near two minutes (the oracle
    # does ~6e4 tet cell-updates/s on 16 host cores; its cost per cell does not depend on the size)
    if args.workload in ("c2", "c5"):
        cells_budget = 120.0 * 6e4 / max(1, args.steps + args.warmup)
        Ns = int(max(8, min(24, (cells_budget / 6.0) ** (1.0 / 3.0))))
    else:
        cells_budget = 120.0 * 1.5e4 / max(1, args.steps + args.warmup)
        per_n3 = 60.0 if args.workload == "c3h" else 12.0  # cells per N^3 of the sphere family
        Ns = int(max(4, min(10, (cells_budget / per_n3) ** (1.0 / 3.0))))
    mi, Q0, ocfg, what = oracle_problem(args.workload, Ns)
    m = O.OracleMesh(mi)
    s = O.OracleSolver(m, Q0, ocfg, threads=threads)
    s.step(args.warmup)
    t0 = time.perf_counter()
    s.step(args.steps)
    dt = time.perf_counter() - t0
    value = m.n_cells * args.steps / dt
    config, scaling, _ = workload_config(args.workload, world, args.box, args.jitter)
    sample = f"each step: one full S2O4 step of the oracle on the {what} (same per-cell work as the workload)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mesh generators and initial states, workloads.py)",
            "config": config,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--workload", default="c5", choices=["c2", "c3", "c4", "c5", "c3h"],
                    help="c5: 110^3 Kuhn box (7,986,000 tets) per GPU (default: configs[4], the largest "
                         "single-GPU config, weak scaling); c2: 48^3 Kuhn box per GPU (configs[1]); c3: subsonic "
                         "sphere 12x35^3 hexes (configs[2]); c4: supersonic sphere 12x70^3 hexes (configs[3])")
    ap.add_argument("--box", type=int, default=0,
                    help="c2: cubes per axis per GPU (default 48; SURVEY 8(d) also quotes N = 80)")
    ap.add_argument("--jitter", type=float, default=0.0,
                    help="c2/c5: interior node jitter U[-j h, j h] (seed 656), SURVEY 8(d) benchmark rule")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="halo exchange for --gpus > 1: NCCL send/recv (default) or the fused NVLink put (f3; EXPERIMENTAL: its cross-process flag protocol has not run on a multi-GPU node yet)")
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32],
                    help="64: the fp64 path BASELINE's metric names (default); 32: the FP32 variant (P:1098-1183)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and "OMP_NUM_THREADS" not in os.environ:
        # every rank builds its own region of the mesh on the host (OpenMP): share the cores
        os.environ["OMP_NUM_THREADS"] = str(max(1, len(os.sched_getaffinity(0)) // world))
    import torch
    import torch.distributed as dist
    from paper_2407_00656_b200 import hgks, workloads as W

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    config, scaling, layout = workload_config(args.workload, world, args.box, args.jitter)
    if args.workload in ("c2", "c5"):
        nx, ny, nz = config["box_cubes"]
        mi = W.kuhn_box(nx, ny, nz, h=2.0 / config["block_cubes"], jitter=args.jitter)
        Q0 = W.advection_ic(mi, gamma=GAMMA)
        cfg = hgks.SolverConfig(gamma=GAMMA, cfl=CFL, precision=args.precision)
    else:
        ma, re, n = SPHERE[args.workload]
        mi = sphere_mesh(args.workload, n)
        fs = (1.0, ma, 0.0, 0.0, 1.0 / GAMMA)
        Q0 = W.uniform_state(mi.n_cells, 1.0, (ma, 0.0, 0.0), 1.0 / GAMMA, gamma=GAMMA)  # free-stream IC
        cfg = hgks.SolverConfig(gamma=GAMMA, cfl=sphere_cfl(args.workload), tau_mode=1, mu_inf=ma / re, c1=1.0, t_inf=1.0 / GAMMA,
                                freestream=fs, precision=args.precision)
    # one process per GPU: each builds only its own region (O(owned + ghosts) host setup)
    mesh = hgks.Mesh(mi, n_ranks=world, rank=rank if world > 1 else None)
    nid = None
    if world > 1:
        obj = [hgks.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    tr = hgks.TRANSPORT_P2P if (world > 1 and args.transport == "p2p") else hgks.TRANSPORT_NCCL
    s = hgks.Solver(mesh, Q0, cfg, device=local, rank=rank, nccl_id=nid, transport=tr)
    if tr == hgks.TRANSPORT_P2P:
        s.p2p_connect_dist()
    info = mesh.info(rank)
    n_owned = info["n_owned"]
    stream = s.stream

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    # ---------------- warm-up ----------------
    s.step(args.warmup, info=False)
    s.step(1, info=False)  # captures the step graph (single rank) outside the timed region
    barrier()
    # ---------------- timed region: K steps as a user runs them (CUDA-graph replays on one
    # rank, no per-kernel events), device time by CUDA events on the solver stream ----------------
    launches0 = s.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        s.step(args.steps, info=False)
        ev1.record(stream)
        barrier()
    launches = s.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    # ---------------- profiled pass (every launch bracketed by events): per-kernel times ----------------
    s.set_profiling(True)
    evA, evB = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    evA.record(stream)
    s.step(args.steps, info=False)
    evB.record(stream)
    barrier()
    ms_prof = evA.elapsed_time(evB)
    s.set_profiling(False)
    ktimes = s.kernel_times()
    st = s.step(0)  # sync + positivity check
    t_ms = torch.tensor([ms], dtype=torch.float64, device="cuda")
    tot_cells = torch.tensor([n_owned], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_cells, op=dist.ReduceOp.SUM)
    ms_max = float(t_ms.item())
    cells = float(tot_cells.item())
    value = cells * args.steps / (ms_max * 1e-3)

    # ---------------- end to end through the public API with host buffers ----------------
    # Pipelined through the C-ABI: step k+1's H2D and step k's D2H run on the library's
    # copy streams while neighbouring steps compute (hgks_set_state / hgks_get_state_async).
    Qh = torch.from_numpy(np.ascontiguousarray(Q0)).pin_memory()
    outs = [torch.empty((n_owned, 5), dtype=torch.float64).pin_memory() for _ in range(2)]
    e2e_steps = max(1, args.e2e_steps)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_steps):
        s.set_state(Qh, 0.0)          # H2D of this step's inputs
        s.step(1, info=False)
        s.get_state_async(outs[i % 2])  # D2H of the step's result
    s.sync()                          # the solver stream has waited for every copy
    e1.record(stream)
    e1.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = cells * e2e_steps / (float(e2e_ms.item()) * 1e-3)
    h2d = (mi.n_cells if world == 1 else n_owned) * 5 * 8
    d2h = n_owned * 5 * 8

    # ---------------- roofline of the dominant kernel ----------------
    hbm_peak, hbm_src, alu_peak, alu_src = peaks(args.precision)
    flops = json.load(open(os.path.join(ROOT, "profiles", "flops_per_unit.json")))
    flops_alg = json.load(open(os.path.join(ROOT, "profiles", "flops_algorithmic.json")))

    def roof_of(name):
        kt = ktimes[name]
        if kt["launches"] == 0 or kt["ms"] <= 0:
            return None
        avg_ms = kt["ms"] / kt["launches"]
        if name.startswith("k_recon"):
            # recon runs over owned cells and layer-1 ghosts
            n_recon = info["n_owned"] + info["ghost_layer"][0]
            bytes_per_launch = recon_bytes_per_cell(*layout, rs=args.precision // 8) * n_recon
            achieved = bytes_per_launch / (avg_ms * 1e-3) / 1e9
            return {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": None,
                    "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
                    "peak_source": hbm_src + " (burst copy)"}
        fkey = "c2" if args.workload == "c5" else args.workload  # same tet kernels and per-face work
        nf = info["n_faces"] - info["n_faces_bc"]  # interior faces (the counts are per interior face)
        # algorithmic flops where counted (tau = 0 flux), else the executed SASS count (labelled)
        fpf = flops_alg.get(args.workload, {}).get(name, {}).get(f"fp{args.precision}_flops_per_face")
        src = ("algorithmic: plain evaluation of SURVEY A.10 with an op-counting scalar, "
               "profiles/flops_algorithmic.json (tools/flop_count)")
        if not fpf:
            fpf = flops.get(fkey, {}).get(name, {}).get(f"fp{args.precision}_flops_per_face")
            src = "executed: ncu sass op counts (2 fma + add + mul), profiles/flops_per_unit.json"
        if not fpf:
            return None
        if layout[2] == 7:  # hybrid layouts: one interior launch per face kind per stage
            avg_ms *= 2
        achieved = fpf * nf / (avg_ms * 1e-3) / 1e12
        return {"kernel": name, "bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": achieved / alu_peak, "traffic": None, "avg_launch_ms": avg_ms,
                "flops_per_face": fpf, "flops_source": src, "peak_source": alu_src}

    top = max(ktimes.items(), key=lambda kv: kv[1]["ms"])
    roof = roof_of(top[0])
    # the same figures for every reconstruction and flux kernel (north_star: both >= 0.5)
    rooflines = {n: {k: r[k] for k in ("bound", "achieved", "unit", "frac", "avg_launch_ms")}
                 for n in sorted(ktimes) if n.startswith(("k_recon", "k_flux")) for r in [roof_of(n)] if r}
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    if roof and os.path.exists(traffic_path):
        tr = (json.load(open(traffic_path)).get(roof["kernel"])
              if args.workload in ("c2", "c5") and args.precision == 64 else None)
        if tr:
            # ncu DRAM bytes of one launch on the 48^3 box, scaled to this rank's cells
            units = info["n_owned"] + (info["ghost_layer"][0] if roof["kernel"].startswith("k_recon") else 0)
            roof["traffic"] = tr["dram_bytes_per_launch"] * (units / tr["cells"])
            roof["traffic_source"] = "profiles/traffic.json (ncu --set full, one launch)"

    # ---------------- CPU baseline (oracle, rank 0, bounded sample) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.precision == 64:
        cpu = cpu_baseline(args.workload)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "ms_per_step_profiled": ms_prof / args.steps,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64" if args.precision == 64 else "f32",
            "data": "synthetic (seeded mesh generators and initial states, workloads.py)",
            "config": {**config, "cells": int(cells),
                       "parallelism": f"domain decomposition x{world} (RCB, 3 ghost layers, "
                                      f"{'NVLink put' if world > 1 and args.transport == 'p2p' else 'NCCL'})",
                       "l2": "no flush: per-step working set %.2f GB > 126 MB L2" % (mesh.workspace_size(cfg, rank) / 1e9)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "pipelined": True},
            "gpu_launches": launches, "roofline": roof, "rooflines": rooflines, "cpu_baseline": cpu, "clocks": clocks,
            "kernels": {k: {"launches": v["launches"], "avg_ms": v["ms"] / max(1, v["launches"]),
                            "share": v["ms"] / max(1e-30, sum(x["ms"] for x in ktimes.values()))}
                        for k, v in ktimes.items()},
            "fallbacks": st["fallbacks"],
            # context only: the paper's GPU codes ran ~5x (RTX A5000) and ~9x (V100)
            # faster than its 56-core Xeon OpenMP code; here the ratio is to the
            # CPU oracle (a deliberately plain program) on this box's host cores
            "context": {"paper_speedup_vs_56_core_cpu": {"A5000": 5, "V100": 9},
                        "this_run_vs_cpu_oracle": (value / cpu["value"]) if cpu else None},
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
