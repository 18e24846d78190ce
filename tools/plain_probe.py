"""Dev probe: plain CG (C4) and BDDC-PCG histories vs the reference goldens at C2 / C5."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import history_err, golden  # noqa: E402
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402

OPTS = SolverOptions(1e-8, 0.0, 10000, True)
for name in sys.argv[1:] or ["c2", "c5"]:
    g = golden(name)
    if name == "c2":
        p = Problem.poisson(800, 8)
    else:
        cx, cy, kx, ky, dm, ks, seed = (int(v) for v in g["config"])
        p = Problem.poisson(cx, kx, cy, ky, kappa_decades=dm / 1000.0, kappa_seed=ks, rhs_seed=seed)
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), OPTS)
    e = history_err(rep.residual_history, g["pcg_history"])
    xp, rp = pre.pcg(p.rhs(), OPTS, precondition=False)
    hp = np.array(rp.residual_history)
    gp = g["plain_history"]
    n = min(hp.size, gp.size)
    rel = np.abs(hp[:n] - gp[:n]) / gp[:n]
    print(name, "bddc", rep.iterations, int(g["pcg_report"][0]), f"{e:.3e}",
          "plain", rp.iterations, int(g["plain_report"][0]), f"max {rel.max():.3e}",
          "at", int(rel.argmax()), "first100", f"{rel[:100].max():.3e}", "first500", f"{rel[:500].max():.3e}",
          flush=True)
