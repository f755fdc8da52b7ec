#!/usr/bin/env python3
"""Benchmark of the B200 V-cycle hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config cfgX] [--replicas] [--no-cpu-baseline]

N = 1 (default): BASELINE config 2, the headline (BASELINE.json configs[1]):
3D [0,1]^3, 256^3 fp64 cells in 16^3 blocks (L=5), sphere c=(.5,.5,.5) R=0.2
with phi=1, phi=0 on the outer faces, g = seeded 1e-2*U[-1,1); setup + GPU
stencil build + FMG, then a STEP is one V-cycle (2+2 GS-RB) over the whole
mesh, replayed as one CUDA graph.  Inputs are synthetic, generated on the host
(configs.py) and resident in HBM when the timed region starts.  The finest
level alone (phi + rhs = 268 MB) exceeds the 126 MB L2, so no explicit L2
flush is needed between steps.

N > 1 (torchrun, one rank per GPU): BASELINE config 5 -- ONE 1024^3 problem
(two spheres at phi_b = +-1, Gaussian g) Morton-partitioned over the ranks
(csrc/dist.h: per-rank blocks + halo in HBM, halo exchange over NCCL inside
the per-rank CUDA graph, coarse tail on rank 0): strong scaling, the time of a
step is the max over ranks.  ``--replicas`` instead runs N independent copies
of the config (weak scaling).  ``--config`` picks another BASELINE config.

``--impl reference`` times the reference's own CPU solver (oracle/_ref,
compiled from /root/reference) on the host's cores for the same config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V-cycle unknowns/sec (fp64) and % of HBM peak; residual reduction/cycle"
UNIT = "unknowns/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def gs_traffic(name):
    """DRAM bytes per launch of the finest GS kernel from the committed ncu
    capture (profiles/r02_gs_traffic.json), for the headline config only."""
    if name != "cfg2":
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_gs_traffic.json")) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        return None


def gs_traffic_source(name):
    if name != "cfg2":
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_gs_traffic.json")) as f:
            d = json.load(f)
        return d.get("source", "profiles/r02_gs_traffic.json (ncu --set full capture of k_gs_stream)")
    except Exception:
        return None


def vcycle_bytes(mesh, N, dim, nu1=2, nu2=2):
    """Algorithmic bytes of one V-cycle:
    B_V = sum_{l=2..L} [(24(nu1+nu2)+32) n_l + 32 n_l/2^D + 32 n_{l-1}] + 16 sum_l leaf_l."""
    NI = N ** dim
    L = mesh.n_levels
    n = [0] + [len(mesh.level_blocks(l)) * NI for l in range(1, L + 1)]
    leaf = [0] + [sum(1 for b in mesh.level_blocks(l) if mesh.is_leaf(b)) * NI
                  for l in range(1, L + 1)]
    B = 0
    for l in range(2, L + 1):
        B += (24 * (nu1 + nu2) + 32) * n[l] + 32 * n[l] / (1 << dim) + 32 * n[l - 1]
    B += 16 * sum(leaf)
    return B


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region by an NVML
    polling thread (every ~2 ms, so even a 50 ms region gets many samples);
    falls back to `nvidia-smi -lms` when NVML is unavailable."""

    BAD = (("hw_slowdown", "HwSlowdown"), ("hw_thermal_slowdown", "HwThermalSlowdown"),
           ("sw_thermal_slowdown", "SwThermalSlowdown"), ("sw_power_cap", "SwPowerCap"),
           ("hw_power_brake_slowdown", "HwPowerBrakeSlowdown"))

    def __init__(self, device, period_s=None):
        self.device = device
        self.period_s = float(os.environ.get("PMG_CLOCK_POLL_S", "0.0005")) if period_s is None else period_s
        self.sm, self.max_mhz, self.reasons = [], None, set()
        self._stop = None
        self.proc = None
        self._nv = None
        try:  # NVML initialised before the timed region so the first sample is immediate
            self._nv = self._nvml_handle()
        except Exception:
            self._nv = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        idx = self.device
        ids = [x for x in vis.split(",") if x.strip()]
        if ids and all(x.strip().isdigit() for x in ids) and self.device < len(ids):
            idx = int(ids[self.device])
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def __enter__(self):
        import threading
        try:
            if self._nv is None:
                raise RuntimeError("no NVML")
            nv, h = self._nv
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
            bits = {name: getattr(nv, "nvmlClocksEventReason" + suf,
                                  getattr(nv, "nvmlClocksThrottleReason" + suf, 0))
                    for name, suf in self.BAD}
            self._stop = threading.Event()

            def poll():
                while not self._stop.is_set():
                    try:
                        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        r = get_r(h)
                        self.reasons.update(n for n, bit in bits.items() if bit and (r & bit))
                    except Exception:
                        pass
                    self._stop.wait(self.period_s)

            self._th = threading.Thread(target=poll, daemon=True)
            self._th.start()
        except Exception:
            self._stop = None
            try:
                q = ("clocks.sm,clocks.max.sm,clocks_throttle_reasons.hw_slowdown,"
                     "clocks_throttle_reasons.hw_thermal_slowdown,"
                     "clocks_throttle_reasons.sw_thermal_slowdown,clocks_throttle_reasons.sw_power_cap")
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                     "--format=csv,noheader,nounits", "-lms", "20"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.proc = None
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._th.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for line in out.splitlines():
                f = [x.strip() for x in line.split(",")]
                try:
                    self.sm.append(float(f[0]))
                    self.max_mhz = float(f[1])
                except (ValueError, IndexError):
                    continue
                for (name, _), v in zip(self.BAD, f[2:6]):
                    if v.lower() == "active":
                        self.reasons.add(name)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def time_plan_cycles(torch, dev, sol, mesh, case, stream, steps, barrier=None):
    """Device time of `steps` V-cycles OF THE CONFIG'S PLAN (e.g. config 2: the
    8 V-cycles that follow the FMG cycle): passes of at most case.v_cycles
    back-to-back cycles, each pass right after the plan's start -- phi = 0 with
    the pins applied, then the FMG cycle where the plan has one -- which is
    rebuilt outside the timed region.  CUDA events bracket every pass on the
    launching stream (device idle and synchronised on both sides); the pass
    times are summed.  Cycles beyond the plan run on a converged solution,
    where the coarse BiCGStab solves for round-off noise and needs a third more
    iterations (profiles/r02_cycle_by_cycle.txt): they are reported separately
    (`converged_state`), not as the step time.
    Returns (total ms, last CycleStats, max residual after a full pass or None)."""
    import numpy as np
    from paper_2205_09411_b200.mesh import VAR_PHI
    from paper_2205_09411_b200.solver import LAYOUT_INTERIOR
    zeros = np.zeros((mesh.n_blocks, case.N ** case.dim))
    L = mesh.n_levels
    total, done, stats, full_pass_resid = 0.0, 0, None, None
    while done < steps:
        n = min(case.v_cycles, steps - done)
        dev.set_field(VAR_PHI, zeros, layout=LAYOUT_INTERIOR)
        for l in range(1, L + 1):
            sol.apply_pins(l)
        sol.set_have_guess(False)
        torch.cuda.synchronize()
        if barrier:
            barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if case.fmg_first:
            sol.fmg_cycle_async()  # untimed: e0 is recorded behind it on the stream
        e0.record(stream)
        for _ in range(n):
            sol.v_cycle_async()
        e1.record(stream)
        stats = sol.cycle_result()
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
        if n == case.v_cycles:
            full_pass_resid = stats.max_resid
        done += n
    return total, stats, full_pass_resid


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_config(case, mesh):
    """The config dict of a bench line -- identical in both arms (the problem,
    not how an arm decomposes it; that is the line's "parallelism")."""
    step = "one V-cycle after the FMG cycle" if case.fmg_first else "one V-cycle (10 V from phi = 0 is the plan)"
    L = mesh.n_levels
    n_fine = len(mesh.level_blocks(L)) * case.N ** case.dim
    return {"workload": f"{case.name}: {case.notes}; step = {step}", "leaf_cells": case.leaf_cells(mesh),
            "levels": L, "blocks": mesh.n_blocks,
            "l2_flush": f"none needed: the finest level's phi + rhs ({2 * 8 * n_fine / 1e6:.0f} MB) exceed "
                        "the 126 MB L2"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference_run(case, steps, warmup, budget_s=None, threads=None):
    """The reference's own MgSolver (oracle/_ref/libpmgref.so) on host cores."""
    from oracle.oc import REF_SO, PORT_SO, Oracle
    from paper_2205_09411_b200 import configs as cfgs
    kind = "reference" if os.path.exists(REF_SO) else "port"
    threads = threads or os.cpu_count() or 1
    mesh = case.build_mesh()
    o = Oracle(case.dim, case.N, case.lo[:case.dim], case.hi[:case.dim],
               "ref" if kind == "reference" else "port")
    o.build_uniform(case.levels)
    if case.amr_band > 0:
        o.refine_band(case.lsf.as_descs(), case.amr_band, case.max_level)
    t0 = time.perf_counter()
    o.build_stencils(case.lsf.as_descs(), w_min=case.w_min)
    t_st = time.perf_counter() - t0
    g = case.rhs_fields(mesh)
    o.set_field(1, cfgs.padded_from_interior(g, case.dim, case.N))
    o.solver_create(threads=threads)
    if case.fmg_first:
        o.fmg_cycle()
    times = []
    t_start = time.perf_counter()
    for k in range(warmup + steps):
        t = time.perf_counter()
        o.v_cycle()
        dt = time.perf_counter() - t
        if k >= warmup:
            times.append(dt)
        if budget_s and time.perf_counter() - t_start > budget_s and len(times) >= 3:
            break
    leaf = case.leaf_cells(mesh)
    return dict(kind=kind, threads=threads, times=times, leaf=leaf, stencil_s=t_st)


def run_reference(args, case):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    # a bounded sample: at most ~90 s of V-cycles (config 5 at 1024^3 takes ~6 s each on 16 cores)
    r = cpu_reference_run(case, args.steps, args.warmup, budget_s=90.0)
    t = sum(r["times"])
    k = len(r["times"])
    value = r["leaf"] * k / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": k, "warmup": args.warmup, "ms_per_step": 1e3 * t / k, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(case, case.build_mesh()),
        "parallelism": f"host threads x{r['threads']} ({cpu_model()})",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"], "kind": r["kind"],
                         "sample": f"{k} V-cycles of {case.name} after FMG "
                                   f"(median {1e3 * statistics.median(r['times']):.1f} ms)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args, case):
    """ONE problem Morton-partitioned over the torchrun ranks (
    distributed.DistributedMgSolver over csrc/dist.h): each rank holds its
    blocks and their halo, runs its part of every V-cycle as one CUDA graph
    with the NCCL halo exchange captured in it; the coarse tail runs on rank 0.
    Strong scaling: value = the problem's unknowns x steps / (max over ranks of
    the CUDA-event time)."""
    import torch
    import torch.distributed as dist

    from paper_2205_09411_b200 import DeviceMesh, MgConfig, StencilBuildConfig, build_stencils
    from paper_2205_09411_b200.distributed import DistributedMgSolver
    from paper_2205_09411_b200.mesh import VAR_RHS
    from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t0 = time.perf_counter()
    mesh = case.build_mesh()
    t_mesh = time.perf_counter() - t0
    dev = DeviceMesh(mesh, device=local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    t_stencil = time.perf_counter() - t0
    # every rank generates the right-hand side of its own blocks only (the
    # generator is counter-based: the values do not depend on who draws them)
    only = None
    if ws > 1:
        from paper_2205_09411_b200.distributed import owner_of_blocks
        from paper_2205_09411_b200.partition import morton_partition
        only = owner_of_blocks(mesh, morton_partition(mesh, ws)) == rank
    dev.set_field(VAR_RHS, case.rhs_fields(mesh, only=only), layout=LAYOUT_INTERIOR)
    sol = DistributedMgSolver(dev, MgConfig(), world=ws, rank=rank)
    stream = torch.cuda.ExternalStream(dev.stream, device=local)
    L = mesh.n_levels

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # the config's plan (10 V from phi = 0 for config 5): residual history
    hist = [sol.v_cycle().max_resid for _ in range(case.v_cycles)]
    red = [hist[i] / hist[i + 1] for i in range(len(hist) - 1) if hist[i + 1] > 0]
    reduction = math.exp(sum(math.log(x) for x in red) / len(red)) if red else None
    for _ in range(args.warmup):
        sol.v_cycle_async()
    sol.cycle_result()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            sol.v_cycle_async()
        e1.record(stream)
        stats = sol.cycle_result()
        torch.cuda.synchronize()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    # end to end through the public API: K cycles with the stats read back
    # every step (host wall clock); the rank's rhs stays resident
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sol.v_cycle()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    leaf = case.leaf_cells(mesh)
    ms_step = ms_total / args.steps
    peak, peak_kind = measured_peaks()
    BV = vcycle_bytes(mesh, case.N, case.dim)
    vc_gbs = BV / (ms_step * 1e-3) / 1e9
    fbytes = max_over_ranks(sol.field_bytes())
    info = sol.info()
    kernels = info["graph_kernels"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": leaf * args.steps / (ms_total * 1e-3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(case, mesh),
            "parallelism": (f"one problem Morton-partitioned over {ws} GPUs (split level {info['split_level']})"
                            if ws > 1 else "1 GPU (the partitioned path, one rank)"),
            "vcycle_roofline": {"algorithmic_bytes": BV, "achieved": vc_gbs, "peak": peak * ws, "unit": "GB/s",
                                "frac": vc_gbs / (peak * ws), "bytes_per_unknown": BV / leaf,
                                "peak_kind": f"{peak_kind}, x {ws} GPUs"},
            "e2e": {"value": leaf * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 16 + 16 + 4,
                    "mode": "public API per step (DistributedMgSolver.v_cycle: graph launch + stats read, "
                            "host wall clock, max over ranks); rhs resident"},
            "gpu_launches": kernels * args.steps,
            "kernels_per_step_rank0": kernels,
            "transport": {0: "none", 1: "nccl", 2: "in-process"}[info["transport"]],
            "cycle_graph": bool(info["graph"]),
            "field_bytes_per_rank_max": fbytes,
            "halo_cells_per_level_sweep_rank0": info["halo_cells"],
            "clocks": clk.summary(),
            "residual_reduction_per_cycle": reduction,
            "residual_history": hist,
            "setup_s": {"mesh": t_mesh, "stencil_build_gpu": t_stencil},
            "final_max_resid": stats.max_resid,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_b200(args, case):
    import torch
    from paper_2205_09411_b200 import (DeviceMesh, MgConfig, MgSolver, StencilBuildConfig,
                                       build_stencils)
    from paper_2205_09411_b200.mesh import VAR_RHS
    from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_id = local
    torch.cuda.set_device(dev_id)

    t0 = time.perf_counter()
    mesh = case.build_mesh()
    t_mesh = time.perf_counter() - t0
    dev = DeviceMesh(mesh, device=dev_id)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
    t_stencil = time.perf_counter() - t0
    g = case.rhs_fields(mesh)
    dev.set_field(VAR_RHS, g, layout=LAYOUT_INTERIOR)
    sol = MgSolver(dev, None, MgConfig())
    L = mesh.n_levels
    stream = torch.cuda.ExternalStream(dev.stream, device=dev_id)

    r0 = sol.measure_residual().max_resid
    hist = [r0]
    t_fmg = None
    if case.fmg_first:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sol.fmg_cycle_async()
        e1.record(stream)
        hist.append(sol.cycle_result().max_resid)
        t_fmg = e0.elapsed_time(e1)
    for _ in range(case.v_cycles):  # the config's own plan: FMG + 8 V
        hist.append(sol.v_cycle().max_resid)
    plan_v = hist[-case.v_cycles - 1:]
    red = [plan_v[i] / plan_v[i + 1] for i in range(len(plan_v) - 1) if plan_v[i + 1] > 0]
    reduction = math.exp(sum(math.log(x) for x in red) / len(red)) if red else None

    # converged state (cycles beyond the plan), reported beside the step time
    for _ in range(max(3, args.warmup)):
        sol.v_cycle_async()
    sol.cycle_result()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        sol.v_cycle_async()
    e1.record(stream)
    sol.cycle_result()
    torch.cuda.synchronize()
    converged_ms = e0.elapsed_time(e1) / args.steps
    converged_coarse_iters = sol.coarse_info()[0]

    # warmup (untimed): W V-cycles of the plan; then the K timed steps
    bar = torch.distributed.barrier if ws > 1 else None
    time_plan_cycles(torch, dev, sol, mesh, case, stream, max(3, args.warmup), bar)
    with ClockSampler(dev_id) as clk:
        ms_total, stats, replay_resid = time_plan_cycles(torch, dev, sol, mesh, case, stream, args.steps, bar)
    plan_coarse_iters = sol.coarse_info()[0]
    if ws > 1:
        torch.distributed.barrier()
    if ws > 1:
        tt = torch.tensor([ms_total], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    leaf = case.leaf_cells(mesh)
    value = leaf * ws * args.steps / (ms_total * 1e-3)

    # dominant kernel: GS-RB half-sweep of the finest level (12 B/cell algorithmic)
    peak, peak_kind = measured_peaks()
    reps = 20
    gs_ms = sol.time_op(0, L, reps)
    n_fine = len(mesh.level_blocks(L)) * case.N ** case.dim
    gs_bytes = 12.0 * n_fine
    gs_gbs = gs_bytes / (gs_ms * 1e-3) / 1e9
    phases = {
        "gs_half_sweep_finest_ms": gs_ms,
        "restrict_finest_ms": sol.time_op(1, L, reps),
        "prolong_finest_ms": sol.time_op(2, L, reps),
        "record_finest_ms": sol.time_op(3, L, reps),
        "coarse_solve_ms": sol.time_op(4, 0, reps),
    }
    BV = vcycle_bytes(mesh, case.N, case.dim)
    vc_gbs = BV / (ms_step * 1e-3) / 1e9

    # end-to-end through the public API: h2d of the step's input (finest-level
    # rhs from pinned host memory) + V-cycle + d2h of the step's result (stats)
    gL = np.ascontiguousarray(g[np.array(mesh.level_blocks(L))])
    pinned = torch.empty(gL.size, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = gL.reshape(-1)
    pin_np = pinned.numpy()
    import ctypes as C
    ptr = C.c_void_p(pinned.data_ptr())

    def e2e_serial_step():
        dev._check(dev.lib.pmg_b200_upload_level_field(dev.h, VAR_RHS, L, ptr, LAYOUT_INTERIOR))
        sol.v_cycle_async()
        return sol.cycle_result()

    def e2e_run(steps):
        """K steps through the public API, double-buffered as a time-stepping
        caller would: step k's rhs is staged (H2D on the copy stream) while step
        k-1's V-cycle runs, committed (scattered into the field) at the start
        of step k; every one of the K uploads and K stats reads is inside the
        timed region (the first upload is not overlapped)."""
        dev._check(dev.lib.pmg_b200_stage_field_async(dev.h, VAR_RHS, L, ptr, LAYOUT_INTERIOR))
        for k in range(steps):
            dev._check(dev.lib.pmg_b200_commit_staged_field(dev.h))
            sol.v_cycle_async()
            if k + 1 < steps:
                dev._check(dev.lib.pmg_b200_stage_field_async(dev.h, VAR_RHS, L, ptr, LAYOUT_INTERIOR))
            sol.cycle_result()

    def timed(fn):
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if ws > 1:
            tt = torch.tensor([dt], device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        return dt

    e2e_run(max(3, args.warmup))
    e2e_s = timed(lambda: e2e_run(args.steps))
    e2e_val = leaf * ws * args.steps / e2e_s
    for _ in range(max(1, args.warmup)):
        e2e_serial_step()
    e2e_serial_s = timed(lambda: [e2e_serial_step() for _ in range(args.steps)])
    e2e_serial_val = leaf * ws * args.steps / e2e_serial_s
    kernels = sol.kernel_count(0)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        r = cpu_reference_run(case, steps=40, warmup=1, budget_s=20.0)
        cpu = {"value": r["leaf"] * len(r["times"]) / sum(r["times"]), "unit": UNIT,
               "cores": r["threads"], "kind": r["kind"], "cpu_model": cpu_model(),
               "sample": f"{len(r['times'])} V-cycles of {case.name} after FMG on the host "
                         f"(reference MgSolver, {r['threads']} threads; median "
                         f"{1e3 * statistics.median(r['times']):.1f} ms/V-cycle)"}
        r1 = cpu_reference_run(case, steps=5, warmup=0, budget_s=10.0, threads=1)
        cpu["threads_1"] = {"value": r1["leaf"] * len(r1["times"]) / sum(r1["times"]), "unit": UNIT,
                            "cores": 1, "sample": f"{len(r1['times'])} V-cycles, median "
                                                  f"{1e3 * statistics.median(r1['times']):.1f} ms/V-cycle"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(case, mesh),
            "parallelism": f"{ws} independent replicas (weak scaling)" if ws > 1 else "1 GPU",
            "roofline": {"bound": "hbm",
                         "kernel": "finest GS-RB half-sweep (k_gs_stream + concurrent k_gs_cut)",
                         "achieved": gs_gbs, "peak": peak, "unit": "GB/s",
                         "frac": gs_gbs / peak, "traffic": gs_traffic(case.name),
                         "traffic_source": gs_traffic_source(case.name),
                         "bytes_per_launch": gs_bytes, "peak_kind": peak_kind},
            "vcycle_roofline": {"algorithmic_bytes": BV, "achieved": vc_gbs, "peak": peak,
                                "unit": "GB/s", "frac": vc_gbs / peak,
                                "bytes_per_unknown": BV / leaf},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(gL.nbytes),
                    "d2h_bytes_per_step": 16 + 16 + 4,
                    "mode": "public API per step: finest rhs H2D from pinned host memory (double-buffered: "
                            "overlaps the previous step's V-cycle) + V-cycle + stats D2H",
                    "serial_value": e2e_serial_val},
            "gpu_launches": kernels * args.steps,
            "kernels_per_step": kernels,
            "timing": {
                "protocol": f"steps are V-cycles of the config's plan ({'FMG + ' if case.fmg_first else ''}"
                            f"{case.v_cycles} V from phi = 0): passes of <= {case.v_cycles} back-to-back "
                            "cycles timed with CUDA events on the launching stream and summed; before every "
                            "pass phi is reset and the plan's start (pins"
                            f"{', FMG cycle' if case.fmg_first else ''}) rebuilt outside the timed region",
                "plan_replay_matches": (replay_resid == plan_v[-1]) if replay_resid is not None else None,
                "coarse_iters_last_plan_cycle": plan_coarse_iters,
                "converged_state": {
                    "ms_per_step": converged_ms, "coarse_iters": converged_coarse_iters,
                    "note": "back-to-back V-cycles on the converged solution (beyond the plan): the coarse "
                            "BiCGStab then solves for round-off noise and runs more iterations"},
            },
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "fmg_ms": t_fmg,
            "residual_reduction_per_cycle": reduction,
            "residual_history": hist,
            "phases_ms": phases,
            "setup_s": {"mesh": t_mesh, "stencil_build_gpu": t_stencil},
            "final_max_resid": stats.max_resid,
        }
        if ws == 1 and not args.no_extras:
            line["extra_configs"] = extra_configs(args)
            line["stencil_build"] = stencil_build_compare(args)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def extra_configs(args, names=("cfg3", "cfg4")):
    """V-cycle throughput of BASELINE configs 3 (AMR, byte model from the
    actual n_l and leaf_l) and 4 (512^3, 32 spheres) on the same GPU."""
    import torch
    from paper_2205_09411_b200 import DeviceMesh, MgConfig, MgSolver, StencilBuildConfig, build_stencils
    from paper_2205_09411_b200 import configs as cfgs
    from paper_2205_09411_b200.mesh import VAR_RHS
    from paper_2205_09411_b200.solver import LAYOUT_INTERIOR
    out = {}
    peak, _ = measured_peaks()
    for name in names:
        case = cfgs.get_case(name)
        mesh = case.build_mesh()
        dev = DeviceMesh(mesh)
        build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
        dev.set_field(VAR_RHS, case.rhs_fields(mesh), layout=LAYOUT_INTERIOR)
        sol = MgSolver(dev, None, MgConfig())
        hist = [sol.v_cycle().max_resid for _ in range(case.v_cycles)]  # the config's plan
        stream = torch.cuda.ExternalStream(dev.stream)
        steps = max(5, args.steps)
        time_plan_cycles(torch, dev, sol, mesh, case, stream, 3)  # warm-up
        ms_total, _, _ = time_plan_cycles(torch, dev, sol, mesh, case, stream, steps)
        ms = ms_total / steps
        leaf = case.leaf_cells(mesh)
        BV = vcycle_bytes(mesh, case.N, case.dim)
        red = [hist[i] / hist[i + 1] for i in range(len(hist) - 1) if hist[i + 1] > 0]
        out[name] = {"workload": case.notes, "leaf_cells": leaf, "ms_per_step": ms,
                     "value": leaf / (ms * 1e-3), "unit": UNIT,
                     "vcycle_roofline": {"algorithmic_bytes": BV, "achieved": BV / (ms * 1e-3) / 1e9,
                                         "peak": peak, "unit": "GB/s", "frac": BV / (ms * 1e-3) / 1e9 / peak,
                                         "bytes_per_unknown": BV / leaf},
                     "residual_reduction_per_cycle": (math.exp(sum(math.log(x) for x in red) / len(red))
                                                      if red else None)}
        del sol, dev
    return out


def stencil_build_compare(args, names=("cfg2", "cfg4")):
    """K5 end to end (pmg_b200_build_stencils: the device build and every
    device table the solver needs) against the reference's build_stencils on
    all host threads, same host, same inputs."""
    from oracle.oc import REF_SO, Oracle
    from paper_2205_09411_b200 import DeviceMesh, StencilBuildConfig, build_stencils
    from paper_2205_09411_b200 import configs as cfgs
    out = {}
    for name in names:
        case = cfgs.get_case(name)
        mesh = case.build_mesh()
        dev = DeviceMesh(mesh)
        ts = []
        for _ in range(2):
            t0 = time.perf_counter()
            build_stencils(dev, case.lsf, StencilBuildConfig(w_min=case.w_min))
            ts.append(time.perf_counter() - t0)
        del dev
        rec = {"gpu_s_first": ts[0], "gpu_s": min(ts)}
        if os.path.exists(REF_SO) and not args.no_cpu_baseline:
            o = Oracle(case.dim, case.N, case.lo[:case.dim], case.hi[:case.dim], "ref")
            o.build_uniform(case.levels)
            t0 = time.perf_counter()
            o.build_stencils(case.lsf.as_descs(), w_min=case.w_min)
            rec["reference_s"] = time.perf_counter() - t0
            rec["reference_threads"] = os.cpu_count()
            rec["speedup"] = rec["reference_s"] / rec["gpu_s"]
            del o
        out[name] = rec
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None,
                    help="BASELINE config (default: cfg2 on one GPU, cfg5 partitioned on several)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra lines (configs 3 / 4 throughput, stencil build vs the reference)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent copies of the config (weak scaling) instead of one partitioned problem")
    ap.add_argument("--partitioned", action="store_true",
                    help="the partitioned path even on one GPU (one rank)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    ws, _, _ = dist_env()
    partitioned = args.partitioned or (ws > 1 and not args.replicas)
    from paper_2205_09411_b200 import configs as cfgs
    case = cfgs.get_case(args.config or ("cfg5" if partitioned and ws > 1 else "cfg2"))
    if args.impl == "reference":
        return run_reference(args, case)
    if partitioned:
        return run_partitioned(args, case)
    return run_b200(args, case)


if __name__ == "__main__":
    sys.exit(main())
