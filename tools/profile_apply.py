"""Profiling driver (dev tool): build a config, warm up, then run a few applies and one
PCG solve on a side stream. Meant to be wrapped by ncu; prints nothing timing-critical."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402


def main():
    k = int(os.environ.get("K", "8"))
    m = int(os.environ.get("M", "100"))
    napply = int(os.environ.get("NAPPLY", "3"))
    import torch

    p = Problem.poisson(k * m, k, rhs_seed=1)
    pre = Preconditioner(p, leaf_size=int(os.environ.get("LEAF", "24")),
                         solve_parts=int(os.environ.get("PARTS", "0")))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rd = torch.tensor(p.rhs(), device="cuda")
    zd = torch.empty_like(rd)
    for _ in range(napply):
        pre.apply_device(rd.data_ptr(), zd.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    if os.environ.get("PCG", "1") == "1":
        x, rep = pre.pcg(p.rhs(), SolverOptions(1e-8, 0.0, 10000, True))
        print("iterations", rep.iterations, "stats", pre.stats())


if __name__ == "__main__":
    main()
