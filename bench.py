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
batched interior solve) timed live with CUDA events on its launching stream during the timed
solves. `cpu_baseline` is the unmodified reference (oracle/_ref/ref_driver, compiled from
/root/reference/proj/src) timed on this box's host cores on one C2 solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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

CELLS = 100  # cells per subdomain side (10,201 dofs for an interior subdomain)
LAYOUTS = {1: (8, 8), 2: (16, 8), 4: (16, 16), 8: (32, 16)}
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
METRIC = "BDDC-PCG time-to-solution & apply GB/s, 2D Poisson, 1/2/4/8 B200 vs CPU ref"
UNIT = "Mdof/s (global dofs / BDDC-PCG time-to-solution, rtol 1e-8)"


def layout(n_gpus: int):
    if n_gpus in LAYOUTS:
        return LAYOUTS[n_gpus]
    return (8 * n_gpus, 8)


def workload(n_gpus: int) -> dict:
    kx, ky = layout(n_gpus)
    return {"workload": f"C2 weak scaling: 2D Poisson Q1, {kx}x{ky} subdomains of {CELLS}x{CELLS} cells "
                        f"(64 per GPU), BDDC-PCG rtol 1e-8, FP64",
            "cells": [kx * CELLS, ky * CELLS], "subdomains": [kx, ky], "subdomains_per_gpu": 64,
            "global_dofs": (kx * CELLS - 1) * (ky * CELLS - 1), "rhs": "study_rhs(n, seed=1)",
            "l2": "inputs larger than L2 (the factor stream of one interior solve is ~458 MB per GPU)",
            "parallelism": f"subdomain blocks x{n_gpus}"}


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


def ref_solve(n_gpus: int, workers: int, steps: int, warmup: int, timeout: int = 1800) -> dict:
    """Time the unmodified reference (oracle/_ref/ref_driver) on the C2 layout for n_gpus:
    Preconditioner(workers) once (untimed), then warmup + steps full PCG solves."""
    if not os.path.exists(REF_DRIVER):
        raise RuntimeError(f"{REF_DRIVER} missing (built by __graft_entry__.build() where /root/reference exists)")
    kx, ky = layout(n_gpus)
    if kx == ky:
        cmd = [REF_DRIVER, "bench", str(kx), str(CELLS), str(workers), str(steps), str(warmup)]
        out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout).stdout
    else:
        # rectangular layouts go through the reference's own bundle ingest (src/bundle.cpp:113-290)
        from paper_2410_14786_b200 import Problem

        with tempfile.TemporaryDirectory() as d:
            manifest = Problem.poisson(kx * CELLS, kx, ky * CELLS, ky, rhs_seed=1).export_bundle(d)
            cmd = [REF_DRIVER, "benchb", manifest, str(workers), str(steps), str(warmup)]
            out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout).stdout
    return json.loads(out.strip().splitlines()[-1])


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    w = workload(args.gpus)
    # bounded sample: a C2 solve of the reference takes ~0.65 s per GPU's worth of subdomains on
    # 16 cores, so the solves run are capped to ~1 minute of CPU work (mean per solve reported)
    steps = max(2, min(args.steps, int(60.0 / (0.7 * args.gpus))))
    warmup = min(args.warmup, 1)
    r = ref_solve(args.gpus, cores, steps, warmup)
    solve_s = r["solve_seconds_mean"]
    value = r["global_dofs"] / solve_s / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": solve_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": w,
            "iterations": r["iterations"], "final_relative_residual": r["final_relative_residual"],
            "setup_seconds": r["setup_seconds"],
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"{warmup}+{steps} full C2 PCG solves (of the requested {args.warmup}+"
                                       f"{args.steps}, capped to ~1 min of CPU work) of the unmodified reference "
                                       f"(oracle/_ref/ref_driver, Preconditioner workers={cores}); setup untimed"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions, lib
    from paper_2410_14786_b200.distributed import survey_8d

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        from paper_2410_14786_b200.distributed import run_distributed_bench

        run_distributed_bench(args, workload(world), layout(world), CELLS)
        return
    dev = local_rank
    torch.cuda.set_device(dev)
    kx, ky = layout(world)
    prob = Problem.poisson(kx * CELLS, kx, ky * CELLS, ky, rhs_seed=1)
    t0 = time.perf_counter()
    pre = Preconditioner(prob, device=dev)
    setup_s = time.perf_counter() - t0
    st = pre.stats()
    n = prob.global_dofs
    b_host = prob.rhs()
    opts = SolverOptions(1e-8, 0.0, 10000, True)
    stream = torch.cuda.Stream(dev)
    b = torch.from_numpy(b_host).to(f"cuda:{dev}")
    x = torch.empty_like(b)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        rep = pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=stream.cuda_stream)
    stream.synchronize()

    # ---- timed region: K device-resident solves (b, x in HBM)
    pre.kernel_times(reset=True)
    pre.set_profile(True)
    clocks = ClockSampler(dev)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    l0 = lib().bddc_kernel_launches()
    gc.disable()  # the PCG loop is host-driven: no interpreter GC pause inside the timed region
    e0.record(stream)
    reps = []
    for _ in range(args.steps):
        reps.append(pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=stream.cuda_stream))
    e1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    launches = lib().bddc_kernel_launches() - l0
    clk = clocks.stop()
    pre.set_profile(False)
    kt = pre.kernel_times(reset=True)
    ms = e0.elapsed_time(e1) / args.steps
    rep = reps[-1]
    if not rep.converged or any(r.iterations != rep.iterations for r in reps):
        raise SystemExit(f"timed solves disagree / did not converge: {[r.iterations for r in reps]}")

    # ---- e2e: the C-ABI call a user makes (host b -> host x), copies inside the timed region
    b_pin = torch.from_numpy(b_host).pin_memory().numpy()
    x_pin = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    for _ in range(max(1, args.warmup // 2)):
        xh, rh = pre.pcg(b_pin, opts, out=x_pin)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        xh, rh = pre.pcg(b_pin, opts, out=x_pin)
    e2e_s = (time.perf_counter() - t0) / args.steps
    it = rh.iterations
    h2d = 8 * n
    d2h = 8 * n + 8 * it + 8 * it + 8 * max(0, it - 1) + 32 * (it + 1)  # x, history, alpha, beta, scalars
    xd = x.cpu().numpy()
    if not np.array_equal(xd, xh):
        raise SystemExit("device-resident and host-buffer solves differ")

    # ---- roofline of the dominant kernel: the batched interior solve
    launch_ms = kt["interior_ms"] / max(1, kt["interior_launches"])
    alg_bytes = st["interior_apply_bytes"] / 2  # mean over the apply's two interior-solve launches
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "interior_solve_traffic.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get("dram_bytes_per_launch")
    apply_ms = kt["apply_ms"] / max(1, kt["applies"])

    # ---- reference CPU path on this box's host cores (bounded sample: one C2 solve)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cores = host_cores()
        try:
            r = ref_solve(world, cores, 1, 0)
            cpu = {"value": r["global_dofs"] / r["solve_seconds_mean"] / 1e6, "unit": UNIT, "cores": cores,
                   "kind": "reference",
                   "sample": f"1 full C2 PCG solve ({r['iterations']} iterations) of the unmodified reference "
                             f"(oracle/_ref/ref_driver, workers={cores}); solve {r['solve_seconds_mean']:.3f} s, "
                             f"setup {r['setup_seconds']:.2f} s untimed"}
        except Exception as e:  # report, never fall back
            cpu = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": n / (ms * 1e-3) / 1e6, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(world),
        "iterations": rep.iterations, "final_relative_residual": rep.final_relative_residual,
        "setup_seconds": setup_s,
        "apply": {"ms": apply_ms, "bytes": st["apply_bytes"], "GBps": st["apply_bytes"] / (apply_ms * 1e-3) / 1e9,
                  "frac": st["apply_bytes"] / (apply_ms * 1e-3) / 1e9 / peak,
                  "vs_survey_8d": survey_8d(apply_ms, peak)},
        "roofline": {"kernel": "interior_solve_kernel", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": alg_bytes, "launch_ms": launch_ms,
                     "launches_timed": kt["interior_launches"]},
        "cpu_baseline": cpu,
        "e2e": {"value": n / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3, "api": "bddc_gpu_pcg (pinned host b and x)"},
        "gpu_launches": launches // args.steps, "gpu_launches_total": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
