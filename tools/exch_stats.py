"""Exchange latency accounting at N > 1 (dev tool; BDDC_EXCH_STATS=1, run under torchrun)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Problem, Preconditioner, SolverOptions  # noqa: E402
from paper_2410_14786_b200.distributed import init  # noqa: E402

rank, world, lr, nid = init()
lay = {2: (16, 8), 4: (16, 16)}[world]
p = Problem.poisson(lay[0] * 100, lay[0], lay[1] * 100, lay[1])
pre = Preconditioner(p, device=lr, dist=(rank, world, nid))
nl, nr, no, l2g = pre.layout()
b = torch.tensor(p.rhs()[l2g], device=f"cuda:{lr}")
x = torch.empty_like(b)
opts = SolverOptions(1e-8, 0.0, 10000, True)
for _ in range(3):
    pre.pcg_device(b.data_ptr(), x.data_ptr(), opts)
torch.cuda.synchronize()
base = pre.solve_profile().reshape(-1, 8).astype(float)
for _ in range(10):
    pre.pcg_device(b.data_ptr(), x.data_ptr(), opts)
torch.cuda.synchronize()
d = pre.solve_profile().reshape(-1, 8).astype(float) - base
names = ["U halo", "p halo", "h iface", "cbuf", "pq", "rr", "rz(+z)", "b.b", "z halo"]
for t, nm in enumerate(names):
    if d[t, 0]:
        print(f"rank {rank} {nm:8s}: n {d[t,0]:5.0f} total {d[t,1]/d[t,0]/1e3:6.2f} us wait {d[t,2]/d[t,0]/1e3:6.2f} us"
              f" | seq {d[t,3]/d[t,0]/1e3:5.2f} red {d[t,4]/d[t,0]/1e3:5.2f} put {d[t,5]/d[t,0]/1e3:5.2f}"
              f" rel {d[t,6]/d[t,0]/1e3:5.2f}", flush=True)
torch.distributed.barrier()
