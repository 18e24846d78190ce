"""Per-solve device times of the C2 bench loop (dev tool: where do outliers come from?)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402

p = Problem.poisson(800, 8, rhs_seed=1)
pre = Preconditioner(p)
stream = torch.cuda.Stream()
b = torch.tensor(p.rhs(), device="cuda")
x = torch.empty_like(b)
opts = SolverOptions(1e-8, 0.0, 10000, True)
pre.set_profile(os.environ.get("PROFILE", "0") == "1")
for _ in range(3):
    pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=stream.cuda_stream)
torch.cuda.synchronize()
for rnd in range(int(os.environ.get("ROUNDS", "5"))):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(31)]
    ev[0].record(stream)
    for i in range(30):
        pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=stream.cuda_stream)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    t = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(30)])
    print(f"round {rnd}: mean {t.mean():.3f} median {np.median(t):.3f} max {t.max():.3f} min {t.min():.3f} "
          f"n>4ms {(t > 4.0).sum()}  {' '.join(f'{v:.2f}' for v in t if v > 4.0)}", flush=True)
