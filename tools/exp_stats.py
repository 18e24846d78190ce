"""Per-warp cycle accounting of the interior solve (dev tool; needs BDDC_SOLVE_STATS=1)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14786_b200 import Preconditioner, Problem
import torch
k, m = int(os.environ.get("K", 8)), int(os.environ.get("M", 100))
p = Problem.poisson(k * m, k)
pre = Preconditioner(p, leaf_size=int(os.environ.get("LEAF", 16)))
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
r = torch.tensor(p.rhs(), device="cuda"); z = torch.empty_like(r)
for _ in range(3): pre.apply_device(r.data_ptr(), z.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
d = pre.solve_profile()   # last launch = second interior solve of the apply
tot, wait, bar, nu = d[:, 0], d[:, 1], d[:, 2], d[:, 3]
print("warps", len(d), "total cycles: mean %.0f max %.0f" % (tot.mean(), tot.max()))
print("wait  mean %.0f (%.0f%%)  bar mean %.0f (%.0f%%)  work mean %.0f (%.0f%%)" % (
    wait.mean(), 100 * wait.mean() / tot.mean(), bar.mean(), 100 * bar.mean() / tot.mean(),
    (tot - wait - bar).mean(), 100 * (tot - wait - bar).mean() / tot.mean()))
print("units per warp: mean %.1f max %d" % (nu.mean(), nu.max()))
w0 = d[:16]
print("CTA0 per warp (total, wait, bar, units):"); print(w0)
