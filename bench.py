#!/usr/bin/env python
"""Benchmark of the fp64 spherical-grid Jacobi-PCG parabolic solve (MAS, arXiv 2303.03398) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 --master-port P bench.py --gpus N

Metric (BASELINE.json): "PCG iterations/s & matvec HBM GB/s (% of peak) at 1/2/4/8 B200".
Workload (BASELINE.json configs[2]): the coronal-relaxation-shaped viscosity
solve on a 150 x 300 x 600 stretched spherical grid (27.0 M cells), tol 1e-10, strong scaling over
phi-slabs.  One STEP = the whole hot path of SURVEY.md 8(a) for one synthetic input: grid/metric
setup (a1), coefficient assembly (a2), boundary conditions, and the PCG solve to 1e-10 (a3-a11).
``value`` = PCG iterations of the global solve per second (one solve spans all ranks).

Rank 0 prints ONE JSON line.  Timing: W untimed steps, then K steps bracketed by barrier +
cuda.synchronize, CUDA events on the launching stream, max over ranks.  The working set
(~2.2 GB) is far larger than the 126 MB L2, so no explicit flush is needed.
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
# Only the JSON line goes to stdout: file descriptor 1 is pointed at stderr for the whole run (NCCL
# and other libraries print e.g. "NCCL version ..." on stdout), and emit() writes to the saved stdout.
_JSON_OUT = None


def emit(line: dict):
    global _JSON_OUT
    if _JSON_OUT is None:
        _JSON_OUT = sys.stdout
    if SHARED_GPU:
        line["test_mode"] = "MASPCG_BENCH_SHARED_GPU: every rank on cuda:0, not a measurement"
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


def protect_stdout():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)

METRIC = "PCG iterations/s & matvec HBM GB/s (% of peak) at 1/2/4/8 B200"
UNIT = "PCG iterations/s"
# Test mode only (MASPCG_BENCH_SHARED_GPU=1, with --comm peer): every torchrun rank on cuda:0 and a gloo
# process group, so the N > 1 code path of this script (slabs, peer communicator, barriers, max over
# ranks, rank-0 output) runs on a one-GPU box.  Never used for a reported number.
SHARED_GPU = os.environ.get("MASPCG_BENCH_SHARED_GPU") == "1"


def init_dist(world):
    import torch
    import torch.distributed as dist
    local = 0 if SHARED_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return local


def max_over_ranks(v, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device="cpu" if SHARED_GPU else dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# algorithmic bytes per cell of each kernel
PATHS = {
    1: {"name": "three kernels", "stencil": ("stencil_matvec_dot (k_matvec_vec2; k_matvec_flat for odd nr)", 48),
        "update": ("update_jacobi_dots (k_update_vec2; k_update for odd nr)", 32), "pupdate": ("x_and_p_update (k_pupdate_vec2; k_pupdate for odd nr)", 48), "iter": 128},
    2: {"name": "fused two passes", "stencil": ("pass A: p-update + x-update + stencil + p.q (k_pass_a)", 80),
        "update": ("pass B: r-update + Jacobi + r.z, r.r (k_pass_b)", 32), "pupdate": None, "iter": 112},
    3: {"name": "wave", "stencil": ("wave: x/p-update + stencil + p.q, flag-ordered (k_wave)", 80),
        "update": ("update_jacobi_dots (k_update_vec2)", 32), "pupdate": None, "iter": 112},
    4: {"name": "single reduction (Chronopoulos-Gear)",
        "stencil": ("cg1 matvec: w = A u, Dot2 w.u (the stencil kernel k_matvec_vec2 on u)", 48),
        "update": ("cg1 update: convergence, p, s, x, r, u = r/D, Dot2 r.u, r.r (k_cg1_update)", 88),
        "pupdate": None, "iter": 136},
    6: {"name": "persistent (one cooperative kernel per chunk, grid barriers)",
        "stencil": ("persistent chunk kernel (k_persist)", 128), "update": ("(inside k_persist)", 0),
        "pupdate": None, "iter": 128},
}


# BASELINE.json configs[i] of each workload name
CONFIG_INFO = {
    "c1": ("configs[0]", "tiny spherical shell, uniform grid, constant coefficient"),
    "c2": ("configs[1]", "nonuniform stretched grid, radially varying thermal-conduction coefficient"),
    "c3": ("configs[2]", "coronal-relaxation-shaped viscosity solve"),
    "c4": ("configs[3]", "weak-scaling per-GPU slab, high-contrast thermal-conduction coefficients"),
    "c5": ("configs[4]", "repeated warm-started implicit solves of a time loop (paper-sized grid)"),
    "c1a": ("configs[0] grid", "field-aligned thermal conduction (SURVEY 8(f) NEXT-4), 19-point operator"),
    "c2a": ("configs[1] grid", "field-aligned thermal conduction (SURVEY 8(f) NEXT-4), 19-point operator"),
    "c3a": ("configs[2] grid", "field-aligned thermal conduction (SURVEY 8(f) NEXT-4), 19-point operator"),
}


def workload(cfg, nr, nt, np_, tol, maxit, shape):
    idx, desc = CONFIG_INFO.get(cfg, ("-", cfg))
    w = f"{cfg} {nr}x{nt}x{np_} {desc} (BASELINE.json {idx})"
    if shape:
        w += " [grid overridden by --shape]"
    return w + (f", tol={tol:g}" if tol > 0 else f", tol=0 maxit={maxit}") + ", Jacobi-PCG fp64"


def make_config(args, nr, nt, np_, tol, maxit, shape, world, par_note=""):
    """The workload description, identical for both arms (ours and --impl reference)."""
    ws = 80 * nr * nt * np_ / max(world, 1)   # Tr, Tt, Tp, D, sV, p, q, r, x, rhs per rank (~10 doubles/cell)
    l2 = (f"no flush: the per-GPU working set ({ws / 1e6:.0f} MB) exceeds the 126 MB L2 between steps"
          if ws > 126e6 else
          f"no flush: the per-GPU working set ({ws / 1e6:.1f} MB) is L2-resident (no HBM roofline claim)")
    return {"workload": workload(args.config, nr, nt, np_, tol, maxit, shape), "global_cells": nr * nt * np_,
            "parallelism": f"phi-slab x{world}" + par_note, "l2": l2}


def step_stats(ms_list):
    a = np.asarray(ms_list, dtype=np.float64)
    if a.size == 0:
        return None
    return {"min": float(a.min()), "median": float(np.median(a)), "mean": float(a.mean()), "max": float(a.max())}


def host_cpu_info():
    """lscpu model / sockets / cores and this process's CPU affinity (the cores the oracle may use)."""
    info = {"affinity_cpus": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=20).stdout
        kv = {}
        for ln in out.splitlines():
            if ":" in ln:
                k, v = ln.split(":", 1)
                kv[k.strip()] = v.strip()
        sockets = int(kv.get("Socket(s)", "0") or 0)
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        info.update({"model": kv.get("Model name"), "sockets": sockets, "cores_per_socket": cps,
                     "threads_per_core": int(kv.get("Thread(s) per core", "0") or 0),
                     "logical_cpus": int(kv.get("CPU(s)", "0") or 0), "physical_cores": sockets * cps or None})
    except Exception as e:   # lscpu missing: affinity only
        info["lscpu_error"] = str(e)
    return info


def omp_threads(info):
    phys = info.get("physical_cores") or info["affinity_cpus"]
    return max(1, min(phys, info["affinity_cpus"]))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({n for s in self.samples for n, v in zip(self.NAMES, s[2:]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def ncu_traffic_per_launch(path_id, name=None):
    """dram__bytes_read.sum + dram__bytes_write.sum of the stencil kernel from the committed
    `ncu --set full` summary of that path (profiles/ncu_stencil_path{1,2}.json, or profiles/<name>.json), or None."""
    path = os.path.join(ROOT, "profiles", f"{name}.json" if name else f"ncu_stencil_path{path_id}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        k = d["kernels"][0]
        return float(k["dram_bytes_per_launch"]), d.get("source", path)
    except Exception:
        return None, None


def oracle_sample(prob, iters: int, openmp: bool = False):
    """Time the CPU oracle (as it stands; single-threaded, or its -fopenmp build on all host cores) on
    the full grid: setup once, then `iters` PCG iterations (tol = 0).  Returns (iterations/s, seconds of
    CPU work, seconds per iteration)."""
    import oracle
    oracle.use_openmp(openmp)
    t0 = time.perf_counter()
    if getattr(prob, "krt", None) is not None:   # field-aligned conduction (NEXT-4)
        op = oracle.AnisoOperator(prob.rf, prob.tf, prob.pf, prob.kr, prob.kt, prob.kp, prob.s, prob.bc_in,
                                  prob.bc_out, prob.krt, prob.krp, prob.ktp)
    else:
        op = oracle.Operator(prob.rf, prob.tf, prob.pf, prob.kr, prob.kt, prob.kp, prob.s, prob.bc_in, prob.bc_out)
    b = op.rhs(prob.f, prob.g_in, prob.g_out)
    t1 = time.perf_counter()
    op.pcg(b, prob.x0, 0.0, 0)
    t2 = time.perf_counter()
    op.pcg(b, prob.x0, 0.0, iters)
    t3 = time.perf_counter()
    oracle.use_openmp(False)
    per_iter = ((t3 - t2) - (t2 - t1)) / iters
    return 1.0 / per_iter, t3 - t0, per_iter


def cpu_baseline_block(prob, cfg, iters1: int, iters_all: int):
    """cpu_baseline: the oracle on all physical host cores (-fopenmp build of the same source:
    per-cell loops threaded, dot products sequential) and single-threaded, on a bounded sample."""
    info = host_cpu_info()
    nth = omp_threads(info)
    os.environ["OMP_NUM_THREADS"] = str(nth)   # read when the -fopenmp library initialises
    ips1, s1, per1 = oracle_sample(prob, iters1, openmp=False)
    ipsn, sn, pern = oracle_sample(prob, iters_all, openmp=True)
    return {"value": ipsn, "unit": UNIT, "cores": nth, "kind": "oracle",
            "sample": f"oracle/masoracle.c built with -fopenmp, OMP_NUM_THREADS={nth} (physical cores in this "
                      f"process's affinity), on the full {cfg} grid: operator assembly + rhs + r0 once, then "
                      f"{iters_all} PCG iterations (tol=0); {sn:.1f} s of CPU work, {pern * 1e3:.0f} ms/iteration",
            "single_thread": {"value": ips1, "cores": 1,
                              "sample": f"plain build, 1 thread, {iters1} PCG iterations; {s1:.1f} s of CPU work, "
                                        f"{per1 * 1e3:.0f} ms/iteration"},
            "host": info}


VV_BYTES = {"matvec": 104, "update": 96, "pupdate": 144, "iter": 344}   # algorithmic B/cell


def oracle_vv_sample(prob, iters: int):
    """Time the vector oracle (as it stands, single-threaded) on the full grid: coefficients, diagonal
    and rhs once, then `iters` PCG iterations (tol = 0).  Returns (iterations/s, CPU seconds, s/iter)."""
    import oracle
    T = lambda g: None if g is None else np.ascontiguousarray(np.transpose(g, (1, 0, 2)))
    t0 = time.perf_counter()
    op = oracle.VVOperator(prob.rf, prob.tf, prob.pf, prob.nu, prob.s, prob.wall_in, prob.wall_out)
    b = op.rhs(prob.f, T(prob.g_in), T(prob.g_out))
    t1 = time.perf_counter()
    op.pcg(b, prob.x0, 0.0, 0)
    t2 = time.perf_counter()
    op.pcg(b, prob.x0, 0.0, iters)
    t3 = time.perf_counter()
    per_iter = ((t3 - t2) - (t2 - t1)) / iters
    return 1.0 / per_iter, t3 - t0, per_iter


def run_vv(args):
    """--operator vv: the staggered vector viscosity solve on the coronal grid of
    c3 (config c3v): per step vv_set_coefficients + vv_set_bc_r + vv_solve to 1e-10."""
    import torch
    import torch.distributed as dist
    from paper_2303_03398_b200 import inputs, maspcg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = init_dist(world)
    dev = torch.device(f"cuda:{local}")
    cfg = args.config if args.config in inputs.VV_CONFIGS else "c3v"
    nr, nt, np_ = inputs.VV_CONFIGS[cfg]
    k0, nloc = inputs.slab_extent(np_, rank, world)
    prob = inputs.make_vv_problem(cfg, k0, nloc)
    tol = 0.0 if args.maxit else prob.tol
    maxit = args.maxit if args.maxit else prob.maxit
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    nu, s, f, x0 = T(prob.nu), T(prob.s), T(prob.f), T(prob.x0)
    S = maspcg.Solver(nr, nt, np_, prob.rf, prob.tf, prob.pf, device=local, chunk=args.chunk,
                      force_comm=args.force_comm)
    S.set_option(maspcg.OPT_ARITH, args.arith)
    S.set_option(maspcg.OPT_PDL, args.pdl)
    S.set_option(maspcg.OPT_DEVICE_LOOP, args.device_loop)
    S.vv_enable()
    x = torch.empty_like(x0)
    stream = torch.cuda.current_stream()

    def step():
        S.vv_set_coefficients(nu, s)
        S.vv_set_bc_r(prob.wall_in, None, prob.wall_out, None)
        x.copy_(x0)
        st, info, hist = S.vv_solve(f, x, tol, maxit)
        if st < 0:
            raise RuntimeError(f"vv solve failed: {st} {info.get('error')}")
        return info["iters"]

    for _ in range(args.warmup):
        step()
    S.set_option(maspcg.OPT_TIMING, args.kernel_timing)
    S.reset_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    iters, step_iters = 0, []
    with ClockSampler(local) as clk:
        evs[0].record(stream)
        for k in range(args.steps):
            it = step()
            iters += it
            step_iters.append(it)
            evs[k + 1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = evs[0].elapsed_time(evs[-1])
    step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    stats = S.stats()
    S.set_option(maspcg.OPT_TIMING, 0)
    if world > 1:
        ms = max_over_ranks(ms, dev)
        t = torch.tensor(step_ms, dtype=torch.float64, device="cpu" if SHARED_GPU else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = t.cpu().tolist()
    sec = ms / 1e3
    value = iters / sec
    ncl = prob.nloc * nt * nr
    peak, peak_src = peaks()
    avg = lambda k: stats[k + "_ms"] / stats[k + "_launches"] if stats[k + "_launches"] else 0.0
    mv_ms = avg("matvec")
    achieved = VV_BYTES["matvec"] * ncl / (mv_ms * 1e-3) / 1e9 if mv_ms > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_vv_matvec.json")) as fh:
            traffic = float(json.load(fh)["kernels"][0]["dram_bytes_per_launch"])
    except Exception:
        pass
    gb = lambda k: VV_BYTES[k] * ncl / (avg(k) * 1e-3) / 1e9 if avg(k) > 0 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "kernel": "vv pole-ring sums + vector stencil + p.q (k_vv_ring + k_vv_march, the plane-marching TMA operator; "
                          "MASPCG_VV_MARCH=0: the two-phase k_vv_terms3 + k_vv_rows2)",
                "algorithmic_bytes_per_launch": VV_BYTES["matvec"] * ncl, "avg_launch_ms": mv_ms,
                "peak_source": peak_src, "share_of_step": avg("matvec") * iters / ms if ms > 0 else None,
                "timed_launches": stats["matvec_launches"]}
    per_kernel = {"update_GBps": gb("update"), "p_update_GBps": gb("pupdate"),
                  "iteration_bytes_per_cell": VV_BYTES["iter"],
                  "iteration_GBps": VV_BYTES["iter"] * ncl * iters / sec / 1e9}
    # end to end through the public API from pinned host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hnu, hs, hf, hx0 = pin(prob.nu), pin(prob.s), pin(prob.f), pin(prob.x0)
        hx = torch.empty_like(hx0).pin_memory()

        def step_host():
            dnu, ds, df = hnu.to(dev, non_blocking=True), hs.to(dev, non_blocking=True), hf.to(dev, non_blocking=True)
            S.vv_set_coefficients(dnu, ds)
            S.vv_set_bc_r(prob.wall_in, None, prob.wall_out, None)
            dx = hx0.to(dev, non_blocking=True)
            st, info, hist = S.vv_solve(df, dx, tol, maxit)
            hx.copy_(dx)
            return info["iters"]

        step_host()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it_h = sum(step_host() for _ in range(args.steps))
        torch.cuda.synchronize()
        th = time.perf_counter() - t0
        e2e = {"value": it_h / th, "unit": UNIT,
               "h2d_bytes_per_step": hnu.numel() * 8 + hs.numel() * 8 + hf.numel() * 8 + hx0.numel() * 8,
               "d2h_bytes_per_step": hx.numel() * 8, "ms_per_step": 1e3 * th / args.steps,
               "api": "pinned host -> device copies + maspcg_vv_set_coefficients + maspcg_vv_solve + device -> host"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ips, cpu_s, per_it = oracle_vv_sample(inputs.make_vv_problem(cfg), max(1, args.ref_iters // 4))
        cpu = {"value": ips, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"oracle/masoracle_vv.c (single-threaded C, -O2) on the full {cfg} grid: coefficients, "
                         f"diagonal, rhs once, then {max(1, args.ref_iters // 4)} PCG iterations (tol=0); "
                         f"{cpu_s:.1f} s of CPU work, {per_it * 1e3:.0f} ms/iteration"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2303_03398_b200/inputs.py make_vv_problem)",
            "config": {"workload": f"{cfg} {nr}x{nt}x{np_} staggered vector viscosity solve (SURVEY 8(f) NEXT-2; "
                                   f"grid and viscosity of BASELINE.json configs[2]), tol={tol:g}, Jacobi-PCG fp64",
                       "global_cells": nr * nt * np_, "unknowns": 3 * nr * nt * np_,
                       "parallelism": f"phi-slab x{world}", "iters_per_solve": iters / args.steps,
                       "chunk": args.chunk, "l2": "no flush: working set ~4 GB >> 126 MB L2",
                       "step": "vv_set_coefficients + vv_set_bc_r + vv_solve to tol"},
            "step_ms": step_stats(step_ms),
            "cell_updates_per_s": nr * nt * np_ * value,
            "roofline": roofline, "per_kernel": per_kernel, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": stats["kernel_launches"], "clocks": clk.summary(),
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on the box's host cores (rank 0 only; other ranks
    exit without work).  Same metric, unit and config as our arm; each step is a bounded sample of that
    workload: PCG iterations (tol = 0) of the oracle's -fopenmp build on all physical cores, on the
    full grid, with the operator assembled once before timing."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2303_03398_b200 import inputs
    info = host_cpu_info()
    nth = omp_threads(info)
    os.environ["OMP_NUM_THREADS"] = str(nth)
    oracle.build()
    oracle.build(openmp=True)
    oracle.use_openmp(True)
    shape = tuple(int(v) for v in args.shape.split(",")) if args.shape else None
    aniso = args.operator == "aniso"
    if aniso:
        args.config = args.config if args.config in inputs.ANISO_CONFIGS else "c3a"
        prob = inputs.make_aniso_problem(args.config, shape=shape)
        op = oracle.AnisoOperator(prob.rf, prob.tf, prob.pf, prob.kr, prob.kt, prob.kp, prob.s, prob.bc_in,
                                  prob.bc_out, prob.krt, prob.krp, prob.ktp)
    else:
        prob = inputs.make_problem(args.config, shape=shape)
        op = oracle.Operator(prob.rf, prob.tf, prob.pf, prob.kr, prob.kt, prob.kp, prob.s, prob.bc_in, prob.bc_out)
    tol = 0.0 if args.maxit else prob.tol
    maxit = args.maxit if args.maxit else prob.maxit
    b = op.rhs(prob.f, prob.g_in, prob.g_out)
    m = args.ref_iters
    for _ in range(args.warmup):
        op.pcg(b, prob.x0, 0.0, 1)
    per_step, t_setup_all = [], 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ts = time.perf_counter()
        op.pcg(b, prob.x0, 0.0, 0)          # the r0 = b - A x0 setup alone (removed below)
        t_setup = time.perf_counter() - ts
        op.pcg(b, prob.x0, 0.0, m)
        te = time.perf_counter()
        per_step.append(1e3 * (te - ts - 2 * t_setup))
        t_setup_all += t_setup
    dt = time.perf_counter() - t0
    # each pcg(m) call repeats the r0 = b - A x0 setup, timed separately and removed
    value = args.steps * m / (dt - 2 * t_setup_all) if dt > 2 * t_setup_all else args.steps * m / dt
    oracle.use_openmp(False)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, paper_2303_03398_b200/inputs.py; SURVEY 8(d) recipe)",
        "config": make_config(args, prob.nr, prob.nt, prob.np, tol, maxit, shape, 1),
        "step_ms": step_stats(per_step),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nth, "kind": "oracle",
                         "sample": f"oracle/masoracle.c built with -fopenmp (per-cell loops threaded, dot products "
                                   f"sequential), OMP_NUM_THREADS={nth}, PCG on the full {args.config} grid: {m} "
                                   f"iterations (tol=0) per step, operator assembled once before timing",
                         "host": info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def self_launch(args) -> bool:
    """`python bench.py --gpus N` (N > 1) outside torchrun: launch the N ranks ourselves with
    torch.distributed.run on 127.0.0.1 (rank 0's stdout is ours, so its JSON line is the only output).
    Refuses (exit 2) when fewer than N GPUs are visible instead of silently running one rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    if not SHARED_GPU:
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but {n} CUDA device(s) visible; refusing to run fewer ranks",
                  file=sys.stderr)
            sys.exit(2)
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init lines (rank count, transports) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr)
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--shape", default=None,
                    help="nr,nt,np override of the config's grid (same recipe), e.g. 150,300,75 = the per-GPU "
                         "phi-slab of c3 at 8 GPUs, for one-GPU projections of the strong-scaling iteration")
    ap.add_argument("--chunk", type=int, default=16)
    ap.add_argument("--maxit", type=int, default=None, help="fixed-iteration mode (tol=0), e.g. for ncu")
    ap.add_argument("--from-fields", action="store_true",
                    help="assemble the coefficients each step on the device from the cell density (NEXT-1): "
                         "kappa = nu rho (arithmetic face means), s = rho / dt")
    ap.add_argument("--sts-stages", type=int, default=0,
                    help="also time RKL2 super-time-steps with this many stages (NEXT-4), 0 = off")
    ap.add_argument("--force-comm", action="store_true",
                    help="N=1 with a one-rank NCCL communicator (the multi-rank code path, halos to itself)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="N > 1 (or --force-comm): NCCL, or the peer-memory communicator (exchanges as kernels "
                         "storing into the peers' workspaces over NVLink, CUDA IPC)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-iters", type=int, default=8)
    ap.add_argument("--path", type=int, default=0,
                    help="0 auto, 1 three kernels, 2 fused two passes, 3 wave, 4 single reduction (Chronopoulos-Gear)")
    ap.add_argument("--pdl", type=int, default=1, help="programmatic dependent launch of the loop kernels")
    ap.add_argument("--fuse-halo", type=int, default=2,
                    help="--comm peer: 1 halo stores in the p-update + wait kernel, 2 + the stencil acquires the "
                         "flags itself, 0 separate push kernel (MASPCG_OPT_FUSE_HALO)")
    ap.add_argument("--kernel-timing", type=int, default=2,
                    help="CUDA events around the hot kernels in the timed region: 2 sampled (the middle slot of "
                         "every graph chunk), 3 sampled (slot 0), 1 every iteration, 0 none")
    ap.add_argument("--device-loop", type=int, default=1,
                    help="1 (default): the whole PCG loop as one CUDA-graph launch with a conditional WHILE node "
                         "(MASPCG_OPT_DEVICE_LOOP; used when kernel timing is off); 0: host chunk loop")
    ap.add_argument("--l2-keep", type=int, default=1,
                    help="1 (default): L2 residency of the loop's most-reused arrays when the slab is small "
                         "(MASPCG_OPT_L2_KEEP auto); 0: off")
    ap.add_argument("--vec", type=int, default=1, help="three-kernel path: 1 16-byte vector kernels (nr even), 0 scalar")
    ap.add_argument("--arith", type=int, default=0, help="0 oracle-identical (Dot2, no FMA), 1 fast (FMA)")
    ap.add_argument("--tma", type=int, default=0, help="fused pass A: 1 TMA-staged (nr even), 0 register batches")
    ap.add_argument("--operator", default="scalar", choices=["scalar", "vv", "aniso"],
                    help="scalar: the 7-point parabolic solve (default); vv: the staggered vector viscosity "
                         "(NEXT-2) on the c3 grid (config c3v); aniso: field-aligned thermal conduction "
                         "(NEXT-4, the 19-point operator) on the c3 grid (config c3a)")
    args = ap.parse_args()
    self_launch(args)
    protect_stdout()
    if args.warmup < 3 and args.maxit is None:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.operator == "vv":
        return run_vv(args)

    import torch
    import torch.distributed as dist
    from paper_2303_03398_b200 import inputs, maspcg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    local = init_dist(world)
    dev = torch.device(f"cuda:{local}")

    # ---- synthetic input of this rank's slab (decomposition-independent generator)
    aniso = args.operator == "aniso"
    if aniso and args.config not in inputs.ANISO_CONFIGS:
        args.config = "c3a"
    nr, nt, np_ = (inputs.ANISO_CONFIGS if aniso else inputs.CONFIGS)[args.config]
    shape = tuple(int(v) for v in args.shape.split(",")) if args.shape else None
    if shape:
        nr, nt, np_ = shape
    if args.config == "c4" and not shape:
        np_ *= world
    k0, nloc = inputs.slab_extent(np_, rank, world)
    if aniso:
        prob = inputs.make_aniso_problem(args.config, k0, nloc, shape=shape)
    else:
        prob = inputs.make_problem(args.config, k0, nloc, nranks=world, shape=shape)
    tol = 0.0 if args.maxit else prob.tol
    maxit = args.maxit if args.maxit else prob.maxit
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    kr, kt, kp, s, f, x0 = (T(a) for a in (prob.kr, prob.kt, prob.kp, prob.s, prob.f, prob.x0))
    krt, krp, ktp = (T(a) for a in (prob.krt, prob.krp, prob.ktp)) if aniso else (None, None, None)

    rho_cells = None
    if args.from_fields:
        rc = inputs.midpoints(prob.rf)
        rho_cells = T(np.broadcast_to(inputs.rho_hydro(rc)[None, None, :], prob.s.shape))
    use_peer = args.comm == "peer" and (world > 1 or args.force_comm)
    S = maspcg.Solver(nr, nt, np_, prob.rf, prob.tf, prob.pf, device=local, chunk=args.chunk,
                      force_comm=args.force_comm and not use_peer, comm="peer" if use_peer else "nccl")
    S.set_option(maspcg.OPT_PATH, args.path)
    S.set_option(maspcg.OPT_ARITH, args.arith)
    S.set_option(maspcg.OPT_TMA, args.tma)
    S.set_option(maspcg.OPT_VEC, args.vec)
    S.set_option(maspcg.OPT_PDL, args.pdl)
    S.set_option(maspcg.OPT_FUSE_HALO, args.fuse_halo)
    S.set_option(maspcg.OPT_L2_KEEP, args.l2_keep)
    S.set_option(maspcg.OPT_DEVICE_LOOP, args.device_loop)
    x = torch.empty_like(x0)
    stream = torch.cuda.current_stream()

    warm = args.config == "c5"      # repeated implicit solves of a time loop
    x.copy_(x0)
    fw = f.clone()
    nstep = [0]

    def step():
        S.set_grid(prob.rf, prob.tf, prob.pf)                         # a1
        if args.from_fields:                                          # a2 from physical fields (NEXT-1)
            S.set_coefficients_from_fields(rho_cells, 1e-3, 2, maspcg.MEAN_ARITHMETIC, rho_cells, 1.0 / 1e-2)
        else:
            S.set_coefficients(kr, kt, kp, s)                         # a2
        if aniso:
            S.set_aniso_coefficients(krt, krp, ktp)                   # field-aligned cross terms (NEXT-4)
        S.set_bc_r(prob.bc_in, None, prob.bc_out, None)
        if warm:
            # the caller's time loop (not the solver path): step 0 solves with the c3-like f from x0;
            # step n >= 1 uses the backward-Euler rhs f = s u^{n-1} (b = s V u^{n-1}) and warm-starts
            # from x0 = u^{n-1}
            if nstep[0] > 0:
                torch.mul(s, x, out=fw)
            nstep[0] += 1
        else:
            x.copy_(x0)
        st, info, hist = S.solve(fw if warm else f, x, tol, maxit)    # a3-a11
        if st < 0:
            raise RuntimeError(f"solve failed: {st} {info.get('error')}")
        return info["iters"]

    for _ in range(args.warmup):
        step()
    if warm:   # the timed steps are the time loop from its start: step 0 cold, steps 1.. warm-started
        x.copy_(x0)
        nstep[0] = 0
    S.set_option(maspcg.OPT_TIMING, args.kernel_timing)
    S.reset_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    iters, step_iters = 0, []
    with ClockSampler(local) as clk:
        evs[0].record(stream)
        for k in range(args.steps):
            it = step()
            iters += it
            step_iters.append(it)
            evs[k + 1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = evs[0].elapsed_time(evs[-1])
    step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    stats = S.stats()
    S.set_option(maspcg.OPT_TIMING, 0)
    if world > 1:
        ms = max_over_ranks(ms, dev)
        t = torch.tensor(step_ms, dtype=torch.float64, device="cpu" if SHARED_GPU else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = t.cpu().tolist()
    sec = ms / 1e3
    value = iters / sec                                 # global solve iterations (strong scaling)
    ncell_local = prob.ncell_local

    # ---- roofline of the dominant kernel (the stencil pass), CUDA events on the launching stream
    peak, peak_src = peaks()
    path = dict(PATHS[stats["path"]])
    if aniso:   # the 19-point field-aligned stencil: p, T_r, T_theta, T_phi, D7, Xrt, Xrp, Xtp, q
        path.update({"name": "three kernels, field-aligned 19-point operator",
                     "stencil": ("aniso stencil + p.q (k_aniso_march, the plane-marching TMA stencil; "
                                 "MASPCG_ANISO_MARCH=0: k_aniso_tma)", 72), "iter": 152})
    st_name, st_bpc = path["stencil"]
    mv_ms = stats["matvec_ms"] / max(stats["matvec_launches"], 1)
    achieved = st_bpc * ncell_local / (mv_ms * 1e-3) / 1e9 if mv_ms > 0 else None
    traffic, traffic_src = ncu_traffic_per_launch(stats["path"], "ncu_aniso_stencil" if aniso else None)
    # sampled timing: average per launch over the timed launches, times the launches of the run
    avg = lambda k: stats[k + "_ms"] / stats[k + "_launches"] if stats[k + "_launches"] else 0.0
    kern_ms = (avg("matvec") + avg("update") + avg("pupdate")) * iters
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": st_name, "path": path["name"],
                "algorithmic_bytes_per_launch": st_bpc * ncell_local,
                "avg_launch_ms": mv_ms, "peak_source": peak_src,
                "share_of_step": avg("matvec") * iters / ms if ms > 0 else None,
                "timed_launches": stats["matvec_launches"],
                "timing": {2: "sampled: every chunk-th iteration (the middle slot of each CUDA-graph chunk)",
                           3: "sampled: every chunk-th iteration (slot 0 of each CUDA-graph chunk)",
                           1: "every iteration", 0: "off"}[args.kernel_timing],
                "traffic_source": traffic_src}

    def gbps(key, bpc):
        n = stats[key + "_launches"]
        return bpc * ncell_local / (stats[key + "_ms"] / n * 1e-3) / 1e9 if n and stats[key + "_ms"] > 0 else None

    per_kernel = {
        "path": path["name"],
        "update_kernel": path["update"][0], "update_GBps": gbps("update", path["update"][1]),
        "p_update_GBps": gbps("pupdate", path["pupdate"][1]) if path["pupdate"] else None,
        "iteration_bytes_per_cell": path["iter"],
        "iteration_GBps": path["iter"] * ncell_local * iters / sec / 1e9,
        "kernels_share_of_step": kern_ms / ms if ms > 0 else None,
    }
    if stats["comm_launches"]:
        # the Fig. 3 analogue (MPI time share): the reductions on the critical path and the
        # halo exchange overlapped with the interior planes, per sampled iteration
        red = stats["comm_ms"] / stats["comm_launches"]
        per_kernel.update({"allreduce_ms_per_iteration": red,
                           "halo_ms_per_iteration": stats["halo_ms"] / stats["comm_launches"],
                           "allreduce_share_of_iteration": red * iters / ms if ms > 0 else None})

    # ---- end to end through the C ABI with HOST buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hkr, hkt, hkp, hs, hf, hx0 = (pin(a) for a in (prob.kr, prob.kt, prob.kp, prob.s, prob.f, prob.x0))
        hx = pin(prob.x0)
        h2d = sum(a.nbytes for a in (hkr, hkt, hkp, hs, hf, hx0))
        d2h = hx.nbytes

        if aniso:
            hx3 = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (prob.krt, prob.krp, prob.ktp)]
            h2d += sum(t.numel() * 8 for t in hx3)

        def step_host():
            S.set_grid(prob.rf, prob.tf, prob.pf)
            S.set_coefficients(hkr, hkt, hkp, hs)                    # maspcg_set_coefficients_host
            if aniso:   # pinned host -> device, then maspcg_set_aniso_coefficients
                S.set_aniso_coefficients(*(t.to(dev, non_blocking=True) for t in hx3))
            S.set_bc_r(prob.bc_in, None, prob.bc_out, None)
            hx[...] = hx0
            st, info, hist = S.solve(hf, hx, tol, maxit)              # maspcg_solve_host
            return info["iters"]

        step_host()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it_h = sum(step_host() for _ in range(args.steps))
        torch.cuda.synchronize()
        th = time.perf_counter() - t0
        if world > 1:
            th = max_over_ranks(th, dev)
        e2e = {"value": it_h / th, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": 1e3 * th / args.steps, "api": "maspcg_set_coefficients_host + maspcg_solve_host"}

    # ---- explicit super-time-stepping of the same operator (NEXT-4): stage throughput
    sts = None
    if args.sts_stages >= 2:
        dt_fe = S.sts_dt_limit()
        ns = args.sts_stages
        tau = 0.9 * (ns * ns + ns - 2) / 4.0 * dt_fe
        u = x0.clone()
        S.sts_step(u, tau, ns)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            S.sts_step(u, tau, ns)
        e1.record(stream)
        torch.cuda.synchronize()
        sms = e0.elapsed_time(e1) / args.steps
        stage_ms = sms / ns
        sts = {"stages": ns, "tau_over_dt_fe": tau / dt_fe, "ms_per_step": sms, "stages_per_s": 1e3 / stage_ms,
               "stage_GBps": 80 * ncell_local / (stage_ms * 1e-3) / 1e9, "bytes_per_cell_per_stage": 80}

    # ---- CPU baseline: the oracle as it stands on this box's host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        full = (inputs.make_aniso_problem(args.config, shape=shape) if aniso
                else inputs.make_problem(args.config, shape=shape))
        cpu = cpu_baseline_block(full, args.config, args.ref_iters, 4 * args.ref_iters)

    if rank == 0:
        par_note = ((" (one-rank peer-memory communicator)" if use_peer else " (one-rank NCCL communicator)")
                    if args.force_comm else (" peer-memory communicator" if use_peer else ""))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if (args.config == "c4" and not shape) else "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2303_03398_b200/inputs.py; SURVEY 8(d) recipe)",
            "config": make_config(args, nr, nt, np_, tol, maxit, shape, world, par_note),
            "run": {"iters_per_solve": iters / args.steps, "chunk": args.chunk,
                    "step": ("set_grid + set_coefficients_from_fields(rho; kappa = 1e-3 rho, s = rho/1e-2) + "
                             "set_bc_r + solve to tol") if args.from_fields else
                            "set_grid + set_coefficients + set_bc_r + solve to tol",
                    "arith": "oracle-identical (no FMA, Dot2 dots)" if args.arith == 0 else "fast (FMA, plain sums)",
                    "l2_keep": "auto (MASPCG_OPT_L2_KEEP)" if args.l2_keep else "off",
                    "loop": "device (conditional WHILE graph)" if (args.device_loop and not args.kernel_timing)
                    else "host chunks (kernel timing events need the host loop)" if args.device_loop else "host chunks"},
            "step_ms": step_stats(step_ms),
            "per_step": [{"iters": int(i), "ms": float(m)} for i, m in zip(step_iters, step_ms)]
            if args.steps <= 64 else None,
            # c5: the time loop from its cold step 0 (warm-started steps after it), end-to-end total
            "time_loop": {"steps": args.steps, "total_ms": ms, "total_iters": iters,
                          "note": "step 0 cold (x0 = 0), steps >= 1 warm-started from the previous solution "
                                  "with f = s u^(n-1)"} if warm else None,
            "cell_updates_per_s": nr * nt * np_ * value,
            "roofline": roofline, "per_kernel": per_kernel, "cpu_baseline": cpu, "e2e": e2e, "sts": sts,
            "gpu_launches": stats["kernel_launches"], "clocks": clk.summary(),
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
