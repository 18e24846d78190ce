"""Dev probe: plain CG (C4) time per solve / per iteration; FIXED=N runs exactly N iterations."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402

fixed = int(os.environ.get("FIXED", "0"))
p = Problem.poisson(800, 8)
pre = Preconditioner(p)
b = p.rhs()
o = SolverOptions(1e-300, 0.0, fixed, False) if fixed else SolverOptions(1e-8, 0.0, 10000, False)
for _ in range(3):
    pre.pcg(b, o, precondition=False)
ts = []
for _ in range(10):
    t = time.perf_counter()
    x, rep = pre.pcg(b, o, precondition=False)
    ts.append(time.perf_counter() - t)
print(os.environ.get("TAG", "default"), rep.iterations, "ms min %.2f med %.2f" % (1e3 * min(ts), 1e3 * np.median(ts)),
      "us/it %.2f" % (1e6 * min(ts) / rep.iterations), flush=True)
