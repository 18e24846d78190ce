"""Dev probe: C2 BDDC-PCG with 2 vs 4 CTAs per subdomain in the interior solve (solve_parts):
parity against the golden history, time per solve, mean interior-solve launch time."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from conftest import golden, history_err  # noqa: E402
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = Problem.poisson(800, 8) if cfg == "c2" else Problem.poisson(2520, 24)
g = golden(cfg)
o = SolverOptions(1e-8, 0.0, 10000, True)
for parts in [int(a) for a in os.environ.get("PARTS", "2,4").split(",")]:
    pre = Preconditioner(p, solve_parts=parts)
    b = torch.tensor(p.rhs(), device="cuda")
    x = torch.empty_like(b)
    s = torch.cuda.Stream()
    for _ in range(3):
        pre.pcg_device(b.data_ptr(), x.data_ptr(), o, stream=s.cuda_stream)
    torch.cuda.synchronize()
    pre.kernel_times(reset=True)
    pre.set_profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        r = pre.pcg_device(b.data_ptr(), x.data_ptr(), o, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    kt = pre.kernel_times(reset=True)
    print(cfg, "parts", parts, "ms/solve %.4f" % (e0.elapsed_time(e1) / 20), "interior launch us %.1f" %
          (1e3 * kt["interior_ms"] / max(1, kt["interior_launches"])), "apply us %.1f" % (1e3 * kt["apply_ms"] / max(1, kt["applies"])),
          "its", r.iterations, "hist err %.2e" % history_err(r.residual_history, g["pcg_history"]), flush=True)
    del pre
