#!/usr/bin/env python
"""bench.py — BDDC-PCG time-to-solution on the C2 weak-scaling workload (BASELINE.json configs[1]).

A "step" is one full BDDC-preconditioned CG solve to rtol 1e-8 (reference `pcg`,
src/pcg.cpp:40-109, with M = Preconditioner::apply, src/study.cpp:111-120; setup excluded
exactly like the reference's `solve_seconds`) of the 2D Q1 Poisson problem with 64 subdomains
of 100x100 cells per GPU: 8x8 subdomains at N=1, 16x8 at N=2, 16x16 at N=4, 32x16 at N=8
(SURVEY.md §8 C2). RHS = study_rhs(n, 1) (src/study.cpp:69-75), synthetic.

value = global dofs / time-to-solution (Mdof/s, whole job, higher is better); ms_per_step is
the time-to-solution itself. `e2e` is the same solve through the C-ABI (bddc_gpu_pcg) with
pinned HOST b and x, copies inside the timed region. `roofline` is the dominant kernel (the
batched interior solve) on this build's own algorithmic bytes, timed live with CUDA events on
its launching stream during the timed solves. `cpu_baseline` is the unmodified reference
(oracle/_ref/ref_driver, compiled from /root/reference/proj/src) timed on this box's host cores
on one solve of the same config.

The other SURVEY.md §8 configs ride in the same line under `extra_configs` (each with its own
time-to-solution, iterations, e2e and cpu_baseline): C4 (the C2 problem by plain CG), C3 (strong
scaling, 6.35M dofs, 24x24 subdomains over the GPUs) and C5 (heterogeneous, 8x8 subdomains over
the GPUs). `--config c3|c4|c5` makes one of them the line itself (and `--impl reference
--config ...` times the reference on it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5] [--no-extra] [--no-cpu-baseline]
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CELLS = 100  # cells per subdomain side at C2 (10,201 dofs for an interior subdomain)
LAYOUTS = {1: (8, 8), 2: (16, 8), 4: (16, 16), 8: (32, 16)}
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
METRIC = "BDDC-PCG time-to-solution & apply GB/s, 2D Poisson, 1/2/4/8 B200 vs CPU ref"
UNIT = "Mdof/s (global dofs / BDDC-PCG time-to-solution, rtol 1e-8)"
UNIT_PLAIN = "Mdof/s (global dofs / plain-CG time-to-solution, rtol 1e-8)"
KAPPA_SEED = 0x5EED  # C5's coefficient generator seed (oracle/gen_golden.py BUNDLES["c5"])

# SURVEY.md §8 configs (BASELINE.json configs[1..4]); configs[0] (C1) is a parity-test case.
CONFIG_DOC = {
    "c2": "C2 weak scaling: 2D Poisson Q1, 64 subdomains of 100x100 cells per GPU, BDDC-PCG rtol 1e-8, FP64",
    "c4": "C4: the C2 problem solved by plain CG (empty preconditioner), rtol 1e-8, FP64",
    "c3": "C3 strong scaling: 2D Poisson Q1, 2520x2520 cells (6,345,361 dofs), 24x24 subdomains split over "
          "the GPUs, BDDC-PCG rtol 1e-8, FP64",
    "c5": "C5 strong scaling: bidomain-style heterogeneous Q1 (kappa log-uniform in [1,100] per element), "
          "352x352 cells, 8x8 subdomains split over the GPUs, BDDC-PCG rtol 1e-8, FP64",
}


def layout(n_gpus: int):
    if n_gpus in LAYOUTS:
        return LAYOUTS[n_gpus]
    return (8 * n_gpus, 8)


LAYOUT_OVERRIDE = None  # --subdomains KXxKY: the C2 / C4 layout (e.g. the N=8 layout 32x16 on 4 GPUs)


def problem_spec(cfg: str, n_gpus: int):
    """(cells_x, kx, cells_y, ky, kappa_decades, kappa_seed) of a config at n_gpus."""
    if cfg in ("c2", "c4"):
        kx, ky = LAYOUT_OVERRIDE or layout(n_gpus)
        return kx * CELLS, kx, ky * CELLS, ky, 0.0, 0
    if cfg == "c3":
        return 2520, 24, 2520, 24, 0.0, 0
    if cfg == "c5":
        return 352, 8, 352, 8, 2.0, KAPPA_SEED
    raise ValueError(cfg)


def make_problem(cfg: str, n_gpus: int):
    from paper_2410_14786_b200 import Problem

    cx, kx, cy, ky, dec, ks = problem_spec(cfg, n_gpus)
    return Problem.poisson(cx, kx, cy, ky, kappa_decades=dec, kappa_seed=ks, rhs_seed=1)


def workload(cfg: str, n_gpus: int) -> dict:
    cx, kx, cy, ky, dec, ks = problem_spec(cfg, n_gpus)
    doc = CONFIG_DOC[cfg]
    if LAYOUT_OVERRIDE and cfg in ("c2", "c4"):
        doc = doc.replace("64 subdomains of 100x100 cells per GPU",
                          f"{kx}x{ky} subdomains of 100x100 cells ({kx * ky // n_gpus} per GPU)")
    w = {"workload": doc, "config": cfg, "cells": [cx, cy], "subdomains": [kx, ky],
         "subdomains_per_gpu": kx * ky / n_gpus, "global_dofs": (cx - 1) * (cy - 1), "rhs": "study_rhs(n, seed=1)",
         "preconditioner": "none (plain CG)" if cfg == "c4" else "BDDC",
         "l2": "inputs larger than L2 (the factor streams of one interior solve exceed 126 MB per GPU)"
               if cfg != "c5" else "C5 is small (123k dofs): its factor streams partly fit L2 (no flush)",
         "parallelism": f"subdomain blocks x{n_gpus}",
         "scaling": "strong" if cfg in ("c3", "c5") else "weak"}
    if dec:
        w["kappa"] = {"decades": dec, "seed": ks}
    return w


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region. start()
    returns once the first sample arrived, so the sampler's start-up (process launch, NVML init)
    never overlaps the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        t0 = time.perf_counter()
        while not self.lines and time.perf_counter() - t0 < 5.0:
            time.sleep(0.01)
        time.sleep(0.1)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ref_solve(cfg: str, n_gpus: int, workers: int, steps: int, warmup: int, timeout: int = 1800) -> dict:
    """Time the unmodified reference (oracle/_ref/ref_driver) on a config: Preconditioner(workers)
    once (untimed; none for plain CG), then warmup + steps full PCG solves."""
    if not os.path.exists(REF_DRIVER):
        raise RuntimeError(f"{REF_DRIVER} missing (built by __graft_entry__.build() where /root/reference exists)")
    cx, kx, cy, ky, dec, ks = problem_spec(cfg, n_gpus)
    flags = ["--plain"] if cfg == "c4" else []
    if kx == ky and cx == cy and not dec:
        cmd = [REF_DRIVER, "bench", str(kx), str(cx // kx), str(workers), str(steps), str(warmup)] + flags
        out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout).stdout
    else:
        # rectangular / heterogeneous problems go through the reference's own bundle ingest
        # (src/bundle.cpp:113-290)
        with tempfile.TemporaryDirectory() as d:
            manifest = make_problem(cfg, n_gpus).export_bundle(d)
            cmd = [REF_DRIVER, "benchb", manifest, str(workers), str(steps), str(warmup)] + flags
            out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout).stdout
    return json.loads(out.strip().splitlines()[-1])


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# rough seconds per reference solve on ~16 host cores, per GPU's worth of work (bounded samples)
REF_SOLVE_S = {"c2": 0.7, "c4": 25.0, "c3": 7.0, "c5": 0.3}


def unit_of(cfg: str) -> str:
    return UNIT_PLAIN if cfg == "c4" else UNIT


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    cfg = args.config
    w = workload(cfg, args.gpus)
    # bounded sample: the solves run are capped to ~1 minute of CPU work (mean per solve reported)
    per = REF_SOLVE_S[cfg] * (args.gpus if cfg in ("c2", "c4") else 1)
    steps = max(1, min(args.steps, int(60.0 / per)))
    warmup = min(args.warmup, 1 if per < 5 else 0)
    r = ref_solve(cfg, args.gpus, cores, steps, warmup)
    solve_s = r["solve_seconds_mean"]
    value = r["global_dofs"] / solve_s / 1e6
    sample = (f"{warmup} warm-up + {steps} timed full {cfg.upper()} solves (the driver asked for {args.warmup}+"
              f"{args.steps}; capped to ~1 min of CPU work) of the unmodified reference (oracle/_ref/ref_driver, "
              f"{'plain CG' if cfg == 'c4' else f'Preconditioner workers={cores}'}); setup untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit_of(cfg), "n_gpus": args.gpus,
            "steps": steps, "warmup": warmup, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": solve_s * 1e3, "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": w,
            "iterations": r["iterations"], "final_relative_residual": r["final_relative_residual"],
            "setup_seconds": r["setup_seconds"],
            "cpu_baseline": {"value": value, "unit": unit_of(cfg), "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": unit_of(cfg), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def cpu_reference(cfg: str, n_gpus: int) -> dict:
    """cpu_baseline object: one bounded reference solve of the config on this box's host cores."""
    cores = host_cores()
    try:
        r = ref_solve(cfg, n_gpus, cores, 1, 0)
        return {"value": r["global_dofs"] / r["solve_seconds_mean"] / 1e6, "unit": unit_of(cfg), "cores": cores,
                "kind": "reference", "iterations": r["iterations"], "ms_per_step": r["solve_seconds_mean"] * 1e3,
                "sample": f"1 full {cfg.upper()} solve ({r['iterations']} iterations) of the unmodified reference "
                          f"(oracle/_ref/ref_driver, {'plain CG' if cfg == 'c4' else f'workers={cores}'}); solve "
                          f"{r['solve_seconds_mean']:.3f} s, setup {r['setup_seconds']:.2f} s untimed"}
    except Exception as e:  # report, never fall back
        return {"value": None, "unit": unit_of(cfg), "cores": cores, "kind": "reference", "sample": f"failed: {e}"}


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(path)) if os.path.exists(path) else {}
    if "hbm_gbs" in peaks:
        return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Dist:
    """World-1 stand-in or the torch.distributed context (max / sum over ranks)."""

    def __init__(self, world: int):
        self.world = world
        self.rank, self.local_rank, self.nid = 0, int(os.environ.get("LOCAL_RANK", "0")), None
        if world > 1:
            from paper_2410_14786_b200.distributed import init

            self.rank, _, self.local_rank, _ = init()

    def fresh_id(self):
        if self.world == 1:
            return None
        from paper_2410_14786_b200.distributed import fresh_nccl_id

        return fresh_nccl_id()

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def reduce(self, vals, op="max"):
        if self.world == 1:
            return [float(v) for v in vals]
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=f"cuda:{self.local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return [float(v) for v in t]


def measure(cfg: str, D: Dist, steps: int, warmup: int, clocks_on: bool = True) -> dict:
    """Set up cfg on this rank's GPU, then time `steps` device-resident solves (b, x in HBM) and
    `steps` end-to-end solves through the C-ABI with pinned host b / x (copies timed)."""
    import numpy as np
    import torch

    from paper_2410_14786_b200 import Preconditioner, SolverOptions, lib

    dev = D.local_rank
    torch.cuda.set_device(dev)
    prob = make_problem(cfg, D.world)
    precondition = cfg != "c4"
    t0 = time.perf_counter()
    if D.world > 1:
        pre = Preconditioner(prob, device=dev, dist=(D.rank, D.world, D.fresh_id()))
        n_local, n_rows, n_owned, l2g = pre.layout()
    else:
        pre = Preconditioner(prob, device=dev)
        n_local = n_rows = prob.global_dofs
        l2g = None
    setup_s = time.perf_counter() - t0
    setup_repeat = None
    setup_repeats = []
    if D.world == 1 and cfg == "c2":
        # further constructions in the same process: the steady-state setup, without the one-time
        # costs of the first (kernel module loads, first device allocations of the process); the
        # median of three, as single host-timed constructions vary by 0.1-0.6 s on the pool's boxes
        for _ in range(3):
            del pre
            t0 = time.perf_counter()
            pre = Preconditioner(prob, device=dev)
            setup_repeats.append(time.perf_counter() - t0)
        setup_repeat = statistics.median(setup_repeats)
    st = pre.stats()
    b_host = prob.rhs()
    opts = SolverOptions(1e-8, 0.0, 10000, True)
    stream = torch.cuda.Stream(dev)
    b = torch.from_numpy(np.ascontiguousarray(b_host if l2g is None else b_host[l2g])).to(f"cuda:{dev}")
    x = torch.empty_like(b)
    torch.cuda.synchronize()
    for _ in range(warmup):
        pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, precondition=precondition, stream=stream.cuda_stream)
    stream.synchronize()

    # ---- timed region: device-resident solves
    pre.kernel_times(reset=True)
    pre.set_profile(precondition)
    clocks = ClockSampler(dev) if clocks_on else None
    if clocks:
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.barrier()
    torch.cuda.synchronize()
    l0 = lib().bddc_kernel_launches()
    gc.disable()  # the PCG loop is host-driven: no interpreter GC pause inside the timed region
    e0.record(stream)
    reps = [pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, precondition=precondition, stream=stream.cuda_stream)
            for _ in range(steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    launches = lib().bddc_kernel_launches() - l0
    D.barrier()
    clk = clocks.stop() if clocks else None
    pre.set_profile(False)
    kt = pre.kernel_times(reset=True)
    ms_local = e0.elapsed_time(e1) / steps
    rep = reps[-1]
    ok = rep.converged and all(r.iterations == rep.iterations for r in reps)

    # ---- e2e: the C-ABI call a user makes (host b -> host x), copies inside the timed region
    n = prob.global_dofs
    b_pin = torch.from_numpy(b_host).pin_memory().numpy()
    x_pin = torch.zeros(n, dtype=torch.float64).pin_memory().numpy()
    for _ in range(max(1, warmup // 2)):
        xh, rh = pre.pcg(b_pin, opts, precondition=precondition, out=x_pin)
    torch.cuda.synchronize()
    D.barrier()
    gc.disable()
    t0 = time.perf_counter()
    for _ in range(steps):
        xh, rh = pre.pcg(b_pin, opts, precondition=precondition, out=x_pin)
    e2e_local = (time.perf_counter() - t0) / steps
    gc.enable()
    D.barrier()
    it = rh.iterations
    h2d = 8 * n_local
    d2h = 8 * n_rows + 8 * it + 8 * it + 8 * max(0, it - 1) + 32 * (it + 1)  # x, history, alpha, beta, scalars
    if D.world == 1 and not np.array_equal(x.cpu().numpy(), xh):
        raise SystemExit("device-resident and host-buffer solves differ")

    ms, e2e_s, bad = D.reduce([ms_local, e2e_local, 0.0 if ok else 1.0])
    h2d_t, d2h_t, launches_t = D.reduce([h2d, d2h, launches], op="sum")
    if bad:
        raise SystemExit(f"{cfg}: timed solves disagree or did not converge: {[r.iterations for r in reps]}")
    out = {"cfg": cfg, "n": n, "ms": ms, "e2e_s": e2e_s, "rep": rep, "setup_s": setup_s, "setup_repeat": setup_repeat,
           "setup_repeats": setup_repeats,
           "st": st, "kt": kt,
           "h2d": int(h2d_t), "d2h": int(d2h_t), "launches": int(launches_t), "clk": clk}
    del pre
    torch.cuda.synchronize()
    return out


def kernel_summary(m: dict, peak: float) -> dict:
    """apply and dominant-kernel (interior solve) roofline numbers from the profiled solves."""
    kt, st = m["kt"], m["st"]
    if not kt.get("applies"):
        return {}
    launch_ms = kt["interior_ms"] / max(1, kt["interior_launches"])
    alg_bytes = st["interior_apply_bytes"] / 2  # mean over the apply's two interior-solve launches
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    apply_ms = kt["apply_ms"] / max(1, kt["applies"])
    from paper_2410_14786_b200.distributed import survey_8d

    return {
        "apply": {"ms": apply_ms, "bytes": st["apply_bytes"], "GBps": st["apply_bytes"] / (apply_ms * 1e-3) / 1e9,
                  "frac": st["apply_bytes"] / (apply_ms * 1e-3) / 1e9 / peak,
                  "survey_8d_reference_bytes": survey_8d(apply_ms, peak) if m["cfg"] == "c2" else None},
        "roofline": {"kernel": "interior_solve_kernel", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "alg_bytes_per_launch": alg_bytes,
                     "launch_ms": launch_ms, "launches_timed": kt["interior_launches"]},
    }


def run_ours(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    D = Dist(world)
    peak, peak_src = peak_hbm()
    cfg = args.config
    m = measure(cfg, D, args.steps, args.warmup)
    ks = kernel_summary(m, peak)
    extras = {}
    if not args.no_extra and cfg == "c2":
        for ecfg in ("c4", "c3", "c5"):
            em = measure(ecfg, D, max(3, min(args.steps, 10)), max(1, min(args.warmup, 3)), clocks_on=False)
            ek = kernel_summary(em, peak)
            extras[ecfg] = {
                "workload": workload(ecfg, world), "value": em["n"] / (em["ms"] * 1e-3) / 1e6, "unit": unit_of(ecfg),
                "ms_per_step": em["ms"], "iterations": em["rep"].iterations,
                "final_relative_residual": em["rep"].final_relative_residual, "setup_seconds": em["setup_s"],
                "e2e": {"value": em["n"] / em["e2e_s"] / 1e6, "ms_per_step": em["e2e_s"] * 1e3,
                        "h2d_bytes_per_step": em["h2d"], "d2h_bytes_per_step": em["d2h"]},
                "gpu_launches": em["launches"] // max(3, min(args.steps, 10)),
                "apply_ms": ek.get("apply", {}).get("ms"),
                "roofline_frac": ek.get("roofline", {}).get("frac"),
                "cpu_baseline": None,
            }
    if D.rank != 0:
        D.barrier()
        return
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(cfg, world)
        for ecfg, e in extras.items():
            e["cpu_baseline"] = cpu_reference(ecfg, world)
    else:
        cpu = None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "interior_solve_traffic.json")
    if os.path.exists(prof) and world == 1 and cfg == "c2" and "roofline" in ks:
        traffic = json.load(open(prof)).get("dram_bytes_per_launch")
    rep = m["rep"]
    n, ms = m["n"], m["ms"]
    line = {
        "metric": METRIC, "value": n / (ms * 1e-3) / 1e6, "unit": unit_of(cfg), "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": workload(cfg, world)["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload(cfg, world), "iterations": rep.iterations,
        # steady-state construction (the second in the process); the first one also pays the
        # process's one-time CUDA costs (lazy kernel-module loads, first allocations) and is
        # reported beside it
        "final_relative_residual": rep.final_relative_residual,
        "setup_seconds": m["setup_repeat"] if m["setup_repeat"] is not None else m["setup_s"],
        "setup": {"mode": "device (GPU setup, SURVEY.md §8 f1)", "first_construction_s": m["setup_s"],
                  "repeat_construction_s": m["setup_repeat"], "repeat_constructions_s": m["setup_repeats"], "device_kernels_s": m["st"]["setup_device_seconds"],
                  "setup_classes": m["st"]["unique_subdomains"],
                  "setup_seconds_is": "median of 3 repeat constructions" if m["setup_repeat"] is not None else "first construction"},
    }
    if ks:
        line["roofline"] = dict(ks["roofline"], traffic=traffic, peak_source=peak_src)
        line["apply"] = ks["apply"]
    line.update({
        "cpu_baseline": cpu,
        "e2e": {"value": n / m["e2e_s"] / 1e6, "unit": unit_of(cfg), "h2d_bytes_per_step": m["h2d"],
                "d2h_bytes_per_step": m["d2h"], "ms_per_step": m["e2e_s"] * 1e3,
                "api": "bddc_gpu_pcg (pinned host b and x)" + (" per rank" if world > 1 else "")},
        "gpu_launches": m["launches"] // args.steps, "gpu_launches_total": m["launches"],
        "clocks": m["clk"],
        "extra_configs": extras or None,
    })
    print(json.dumps(line), flush=True)
    D.barrier()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c2", "c3", "c4", "c5"], default="c2",
                    help="SURVEY.md §8 config of the JSON line (c2 = the headline; c2 also reports c3/c4/c5 "
                         "in extra_configs unless --no-extra)")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--subdomains", default=None, help="C2/C4 layout override KXxKY (e.g. 32x16 on 4 GPUs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.subdomains:
        global LAYOUT_OVERRIDE
        LAYOUT_OVERRIDE = tuple(int(v) for v in args.subdomains.lower().split("x"))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
