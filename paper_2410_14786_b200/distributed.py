"""Multi-GPU launch helpers: one process per B200 under torchrun (RANK / LOCAL_RANK /
WORLD_SIZE / MASTER_* from the environment). torch.distributed is only the plumbing that
broadcasts the NCCL unique id and takes the max of the per-rank timings; the solver's own
exchanges (halo, interface, coarse gather, PCG scalars) run inside the native library
(device/comm.cu) on the solve stream.

Reference counterpart: the reference has no multi-process mode; its only parallelism is the
subdomain worker pool (include/bddc/parallel.hpp:19-45). SURVEY.md §8e is the design.
"""
from __future__ import annotations

import os

from .solver import Preconditioner, Problem, dist_unique_id


# the reference-anchored algorithmic bytes of one C2 apply per GPU (64
# subdomains, B_apply = 8·[2F_I + F_S + 2nnz(A) + 2Σ n_local·n_primal + 2n] with the REFERENCE's
# factor counts). Informational only: it credits the algorithmic savings of this build (5.6x
# fewer factor values, no saddle solve), so it is not a roofline fraction of the kernels here;
# bench.py's `roofline.frac` / `apply.frac` use this build's own bytes.
SURVEY_8D_APPLY_BYTES = 1.575e9


def survey_8d(apply_ms: float, peak_gbs: float) -> dict:
    t_roof = SURVEY_8D_APPLY_BYTES / (peak_gbs * 1e9) * 1e3
    return {"bytes": SURVEY_8D_APPLY_BYTES, "reference_roofline_ms": t_roof,
            "reference_bytes_over_apply_time_frac": t_roof / apply_ms}


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
