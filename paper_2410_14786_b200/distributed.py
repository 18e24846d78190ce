"""Multi-GPU launch helpers: one process per B200 under torchrun (RANK / LOCAL_RANK /
WORLD_SIZE / MASTER_* from the environment). torch.distributed is only the plumbing that
broadcasts the NCCL unique id and takes the max of the per-rank timings; the solver's own
exchanges (halo, interface, coarse gather, PCG scalars) run inside the native library
(device/comm.cu) on the solve stream.

Reference counterpart: the reference has no multi-process mode; its only parallelism is the
subdomain worker pool (include/bddc/parallel.hpp:19-45). SURVEY.md §8e is the design.
"""
from __future__ import annotations

import gc
import os
import time

import numpy as np

from .solver import Preconditioner, Problem, SolverOptions, dist_unique_id



# the reference-anchored algorithmic bytes of one C2 apply per GPU (64
# subdomains, B_apply = 8·[2F_I + F_S + 2nnz(A) + 2Σ n_local·n_primal + 2n] with the reference's
# own factor counts) and the target: <= 0.401 ms (60% of the measured-HBM roofline time 0.241 ms).
SURVEY_8D_APPLY_BYTES = 1.575e9


def survey_8d(apply_ms: float, peak_gbs: float) -> dict:
    t_roof = SURVEY_8D_APPLY_BYTES / (peak_gbs * 1e9) * 1e3
    return {"bytes": SURVEY_8D_APPLY_BYTES, "roofline_ms": t_roof, "target_ms": t_roof / 0.6,
            "frac": t_roof / apply_ms, "meets_60pct": apply_ms <= t_roof / 0.6}

def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def fresh_nccl_id() -> bytes:
    """A new NCCL unique id from rank 0, broadcast to every rank (one per communicator:
    ids cannot be reused)."""
    import torch.distributed as dist

    obj = [dist_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def init(backend: str = "nccl"):
    """Initialise torch.distributed (if needed) and return (rank, world, local_rank, nccl_id)."""
    import torch
    import torch.distributed as dist

    rank, world, local_rank = env_rank()
    if backend == "nccl":
        torch.cuda.set_device(local_rank)
    if not dist.is_initialized():
        kw = {"device_id": torch.device(f"cuda:{local_rank}")} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    return rank, world, local_rank, fresh_nccl_id()


def distributed_preconditioner(problem: Problem, **kw) -> Preconditioner:
    """The rank's Preconditioner for a global problem every rank constructed identically."""
    rank, world, local_rank, nid = init()
    return Preconditioner(problem, device=local_rank, dist=(rank, world, nid), **kw)


def run_distributed_bench(args, workload: dict, layout, cells: int) -> None:
    """bench.py at N > 1: weak-scaling C2, every rank solves its block of the global problem."""
    import json

    import torch
    import torch.distributed as dist

    from . import lib

    rank, world, local_rank, nid = init()
    dev = local_rank
    kx, ky = layout
    prob = Problem.poisson(kx * cells, kx, ky * cells, ky, rhs_seed=1)
    t0 = time.perf_counter()
    pre = Preconditioner(prob, device=dev, dist=(rank, world, nid))
    setup_s = time.perf_counter() - t0
    st = pre.stats()
    n_local, n_rows, n_owned, l2g = pre.layout()
    b_host = prob.rhs()
    opts = SolverOptions(1e-8, 0.0, 10000, True)
    stream = torch.cuda.Stream(dev)
    b = torch.from_numpy(np.ascontiguousarray(b_host[l2g])).to(f"cuda:{dev}")
    x = torch.empty_like(b)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        rep = pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=stream.cuda_stream)
    stream.synchronize()

    from bench import ClockSampler  # noqa: E402 (repo root is on sys.path under bench.py)

    pre.kernel_times(reset=True)
    pre.set_profile(True)
    clocks = ClockSampler(dev)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
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
    dist.barrier()
    clk = clocks.stop()
    pre.set_profile(False)
    kt = pre.kernel_times(reset=True)
    ms_local = e0.elapsed_time(e1) / args.steps
    rep = reps[-1]
    ok = rep.converged and all(r.iterations == rep.iterations for r in reps)

    # e2e: host global b -> each rank's block -> host x (C-ABI bddc_gpu_pcg)
    b_pin = torch.from_numpy(b_host).pin_memory().numpy()
    x_pin = torch.zeros(prob.global_dofs, dtype=torch.float64).pin_memory().numpy()
    xh, rh = pre.pcg(b_pin, opts, out=x_pin)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        xh, rh = pre.pcg(b_pin, opts, out=x_pin)
    dist.barrier()
    e2e_local = (time.perf_counter() - t0) / args.steps
    it = rh.iterations
    h2d = 8 * n_local
    d2h = 8 * n_rows + 8 * it + 8 * it + 8 * max(0, it - 1) + 32 * (it + 1)

    t = torch.tensor([ms_local, e2e_local, 0.0 if ok else 1.0, float(h2d), float(d2h), float(launches)],
                     dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_s, bad = float(t[0]), float(t[1]), float(t[2])
    tot = torch.tensor([float(h2d), float(d2h), float(launches)], dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_reduce(tot)
    if bad:
        raise SystemExit("a rank's timed solves disagree or did not converge")
    n = prob.global_dofs
    launch_ms = kt["interior_ms"] / max(1, kt["interior_launches"])
    alg_bytes = st["interior_apply_bytes"] / 2  # mean over the apply's two interior-solve launches
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    import json as _json

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pk = os.path.join(root, "MEASURED_PEAKS.json")
    peaks = _json.load(open(pk)) if os.path.exists(pk) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    apply_ms = kt["apply_ms"] / max(1, kt["applies"])
    if rank == 0:
        from bench import METRIC, UNIT

        line = {
            "metric": METRIC, "value": n / (ms * 1e-3) / 1e6, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload,
            "iterations": rep.iterations, "final_relative_residual": rep.final_relative_residual,
            "setup_seconds": setup_s,
            "apply": {"ms": apply_ms, "bytes": st["apply_bytes"], "GBps": st["apply_bytes"] / (apply_ms * 1e-3) / 1e9,
                      "frac": st["apply_bytes"] / (apply_ms * 1e-3) / 1e9 / peak, "rank": 0,
                      "vs_survey_8d": survey_8d(apply_ms, peak)},
            "roofline": {"kernel": "interior_solve_kernel", "bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)", "alg_bytes_per_launch": alg_bytes,
                         "launch_ms": launch_ms, "rank": 0},
            "cpu_baseline": None,
            "e2e": {"value": n / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(tot[0]),
                    "d2h_bytes_per_step": int(tot[1]), "ms_per_step": e2e_s * 1e3,
                    "api": "bddc_gpu_pcg per rank (pinned host b/x, each rank copies its block)"},
            "gpu_launches": int(tot[2]) // args.steps, "gpu_launches_total": int(tot[2]),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
